// kernels.h — host-side launch wrappers of the sm_100a kernels (kernels.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace minife {

// Device-resident CG scalars of one part (C6).  Written only by CTA 0 of the kernel that
// takes the decision; every CTA computes the same decision from the same exact values.
struct CgState {
    int done;          // a stop test fired (later kernels return immediately)
    int status;        // 0 OK, 6 NOT-SPD, 7 DIVERGED
    int iters;         // completed iterations
    int converged;
    double stop;       // fl(tol * hist[0])
    double pAp, alpha, beta;
};

struct AsmArgs {
    int nx, ny, nz;
    int own_lo[3];
    int64_t own_n[3];
    int64_t rows;                       // owned rows
    int64_t n_ext;
    const int64_t *ext_sorted_gid;      // externals sorted by gid
    const int32_t *ext_sorted_slot;     // their local column (n_owned + slot)
    const int64_t *slice_off;           // [slices+1]
    const uint8_t *row_len;             // [rows]
    int32_t *col;                       // SELL, k-major per slice
    double *val;
    double *b;                          // [rows]
};

struct SpmvArgs {
    int64_t rows, nslices;
    const int64_t *slice_off;
    const uint8_t *row_len;
    const int32_t *col;
    const double *val;
    const double *x;                    // [rows + externals]
    double *y;                          // [rows]
    unsigned long long *acc;            // pAp accumulator (DOT only)
    unsigned long long *acc_zero;       // accumulator to clear (CTA 0), may be null
    const CgState *st;                  // early exit when st->done (may be null)
};

struct UpdArgs {
    int64_t rows;
    double *x, *r, *p;
    const double *Ap;
    const double *b;
    unsigned long long *acc_in;         // finalised at kernel start
    unsigned long long *acc_out;        // accumulated by this kernel
    unsigned long long *acc_zero;       // cleared by CTA 0 (may be null)
    double *hist, *rr;                  // [max_iters+1]
    CgState *st;
};

// Setup (a0.2-a0.5)
cudaError_t launch_rowlen_widths(const AsmArgs &a, uint8_t *row_len, uint8_t *width,
                                 int64_t nslices, cudaStream_t s);
cudaError_t launch_assemble(const AsmArgs &a, cudaStream_t s);

// Hot path
cudaError_t launch_spmv(const SpmvArgs &a, bool with_dot, int grid, cudaStream_t s);
cudaError_t launch_init_vectors(const UpdArgs &a, int grid, cudaStream_t s);
cudaError_t launch_init_finalize(const UpdArgs &a, double tol, cudaStream_t s);
cudaError_t launch_update_xr(const UpdArgs &a, int k, int grid, cudaStream_t s);
cudaError_t launch_update_p(const UpdArgs &a, int k, int grid, cudaStream_t s);

// Halo / virtual transport
cudaError_t launch_pack(const double *src, const int32_t *idx, int64_t n, double *dst,
                        cudaStream_t s);
cudaError_t launch_vsum(unsigned long long *const *accs, int nparts, cudaStream_t s);

// Parity helpers
cudaError_t launch_extract_rows(const int64_t *slice_off, const uint8_t *row_len,
                                const int32_t *col, const double *val, const int64_t *rows,
                                int64_t n, int32_t *out_col, double *out_val,
                                int32_t *out_len, cudaStream_t s);

// occupancy-derived grid sizes
int spmv_grid(int64_t nslices);
int stream_grid(int64_t rows);

constexpr int SPMV_THREADS = 256;
constexpr int UPD_THREADS = 256;

}  // namespace minife
