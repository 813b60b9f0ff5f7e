// api.cu — the C ABI of include/minife.h: context, plans, device buffers, graph-captured CG
// driver, NCCL / virtual-rank transports, parity getters.  Host code; every numeric step of
// the method runs in kernels.cu.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: ranges cost nothing without a profiler

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <string>
#include <vector>

#include "../../include/minife.h"
#include "exact.cuh"
#include "kernels.h"
#include "plan.h"

using namespace minife;

#define MINIFE_VERSION "minife-b200 0.2.0 (sm_100a)"

// ----------------------------------------------------------------------------------------
// NCCL is resolved at run time (dlopen), never linked: the process may already hold torch's
// NCCL (a newer libnccl.so.2 than the system one) and two copies must not be mixed.  Order:
// an already-loaded libnccl.so.2 (RTLD_NOLOAD), then $MINIFE_NCCL_LIB (the binding points it
// at the torch wheel's copy), then the default search path.
// ----------------------------------------------------------------------------------------
namespace {
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommInitAll)(ncclComm_t *, int, const int *);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    const char *(*GetErrorString)(ncclResult_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t);
    ncclResult_t (*Reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int,
                           ncclComm_t, cudaStream_t);
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *);
    ncclResult_t (*CommAbort)(ncclComm_t);
};

const NcclApi *nccl() {
    static NcclApi api;
    static int state = 0;   // 0 untried, 1 ok, -1 failed
    if (state) return state > 0 ? &api : nullptr;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char *env = getenv("MINIFE_NCCL_LIB");
    if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        state = -1;
        return nullptr;
    }
    bool ok = true;
    auto sym = [&](const char *n) {
        void *f = dlsym(h, n);
        if (!f) ok = false;
        return f;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommInitAll = (decltype(api.CommInitAll))sym("ncclCommInitAll");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.Reduce = (decltype(api.Reduce))sym("ncclReduce");
    api.CommGetAsyncError = (decltype(api.CommGetAsyncError))sym("ncclCommGetAsyncError");
    api.CommAbort = (decltype(api.CommAbort))sym("ncclCommAbort");
    state = ok ? 1 : -1;
    return ok ? &api : nullptr;
}

struct Part {
    int dev = 0;
    Plan plan;
    int64_t rows = 0, ncols = 0, nslices = 0, entries = 0, nnz = 0, nns = 0;
    std::vector<int64_t> h_slice_off;
    // matrix (CRS: slice_off/row_len/col/val; SEG: seg/mask/val)
    int64_t *d_slice_off = nullptr;
    uint8_t *d_row_len = nullptr, *d_width = nullptr;
    int32_t *d_col = nullptr, *d_seg = nullptr;
    uint32_t *d_mask = nullptr;
    double *d_val = nullptr;
    // vectors: b, x, r, Ap in row (owned) order; p in column (extended-box) order
    double *d_b = nullptr, *d_x = nullptr, *d_r = nullptr, *d_p = nullptr, *d_Ap = nullptr;
    double *d_p2 = nullptr;                       // fused scheme: second p buffer (lazy)
    double *d_pr[XDEF_MAX] = {};                  // deferred x: ring buffers 2.. (lazy)
    double *d_xin = nullptr, *d_yout = nullptr;   // minife_spmv buffers (lazy)
    // exact accumulators, parity double-buffered: [pAp_0, rr_0, pAp_1, rr_1] x ACC_WORDS
    unsigned long long *d_acc = nullptr;
    int symm_nw = SYMM_NW;                        // SYM SpMV tile width, fixed at assembly
    CgState *d_st = nullptr;
    double *d_hist = nullptr, *d_rr = nullptr;
    double *d_alpha = nullptr;                    // alpha_k history (x every second iteration)
    int hist_cap = 0;
    // halo: send_col = extended columns of the send lists (neighbor order), recv_pos =
    // extended column of each halo slot; wire buffers
    int32_t *d_send_col = nullptr, *d_recv_pos = nullptr;
    int32_t *d_send_row = nullptr;                // send lists as local rows (SYM pre-pack)
    // push transport: per send slot the neighbor index and the receiver's halo column; per
    // neighbor the receiver's p (this device's view: local or peer pointer)
    uint8_t *d_push_nbr = nullptr;
    int32_t *d_push_dst = nullptr;
    double **d_push_ptr = nullptr;
    cudaEvent_t ev_push = nullptr;
    // device-initiated comm (DevComm, kernels.h): this part's comm region, the table of every
    // rank's region as seen from this device, the neighbor ranks; RANK: CUDA-IPC mappings of
    // the other ranks' regions and p arrays (closed on destroy)
    // device comm, halo by r: this part's r-halo receive buffer [externals] (slot order), per
    // send slot the receiver's slot index, per neighbour its r-halo buffer as seen from here
    double *d_rhalo = nullptr;
    int32_t *d_rdst = nullptr;
    double **d_rhalo_ptr = nullptr;
    int32_t *d_tile_order = nullptr;              // SYM SpMV: band-major tile order (or null)
    int64_t tile_order_n = 0;
    unsigned long long *d_comm = nullptr;
    unsigned long long **d_comm_ptrs = nullptr;
    int32_t *d_nbr_rank = nullptr;
    std::vector<void *> ipc_opened;
    double *d_sendbuf = nullptr, *d_recvbuf = nullptr;
    // SEG slice storage order (multi-part): interior slices [0, n_int) first, DESIGN.md §7
    int32_t *d_slice_row = nullptr, *d_slice_pos = nullptr;
    int64_t n_int = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t cstream = nullptr;               // halo transport, overlapped with the SpMV
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;    // per-part timing of assemble / solve
    double t_asm_ms = 0.0, t_solve_ms = 0.0;          // last assemble / solve, this part
    int grid_spmv = 1, grid_upd = 1;
    size_t bytes = 0, matrix_bytes = 0;
    unsigned long long *acc_pAp(int par = 0) const { return d_acc + (2 * (par & 1)) * ACC_WORDS; }
    unsigned long long *acc_rr(int par = 0) const {
        return d_acc + (2 * (par & 1) + 1) * ACC_WORDS;
    }
    double *p_buf(int k) const { return (k & 1) ? d_p2 : d_p; }   // fused: p_k lives in k % 2
    double *ring(int i) const { return i == 0 ? d_p : (i == 1 ? d_p2 : d_pr[i]); }
};

struct DevGuard {
    int prev = 0;
    bool ok = false;
    explicit DevGuard(int dev) {
        ok = cudaGetDevice(&prev) == cudaSuccess;
        cudaSetDevice(dev);
    }
    ~DevGuard() {
        if (ok) cudaSetDevice(prev);
    }
};
// NVTX range per ABI phase (assemble, solve, profile, spmv, verify), visible to Nsight tools
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

struct minife_ctx {
    Mesh mesh{};
    int mode = MINIFE_MODE_SINGLE;
    int fmt = MINIFE_FMT_SEG;
    int scheme = MINIFE_SCHEME_3K;
    int transport = MINIFE_TRANSPORT_DIRECT;   // VIRTUAL ctxs (MULTI: PUSH if peer access)
    bool push_ready = false;                     // push tables built
    int world = 1, rank = 0;
    std::vector<Part> parts;
    cudaStream_t user_stream = nullptr;
    bool assembled = false;
    std::string err;
    // graph cache
    cudaGraphExec_t gexec = nullptr;
    int g_iters = -1;
    double g_tol = -1.0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // timing window (minife_set_timing_window): events around the SpMV launches of
    // iterations [tw_k0, tw_k0 + tw_n) inside the solve itself (graph nodes)
    int tw_k0 = 0, tw_n = 0;
    std::vector<cudaEvent_t> tw_ev;              // [2 * tw_n]: start, end of each SpMV
    bool tw_armed = false;                       // the enqueued solve records the window
    bool eager = false;                          // capture failed once (world > 1): no graphs
    // options (minife_set_option): -1 = automatic choice
    struct {
        int x_defer = -1;          // deferred x update: 0 off, 2..8 forced ring size X
        int small_solver = -1;     // single-launch solvers: 0 none, 1 one CTA, 2 one cluster
        int graph = 1;             // 0: enqueue every solve directly (no CUDA graph)
        int val_evict_first = -1;  // SYM SpMV value stream evict-first in L2
        int x_prefetch = -1;       // SYM SpMV plane-ahead L2 prefetch of x
        int sym_kernel = 1;        // SYM SpMV: 1 tensor-map mirrors, 0 L1-gather kernel
        int spmv_impl = -1;        // SEG/CRS SpMV: 1 TMA pipeline, 0 register streaming
        int x_late = 1;            // x += alpha p applied by K7 (1) or K6 (0)
        int cluster_dd = 1;        // cluster solver: DSMEM digit pushes
        int device_comm = -1;      // MULTI/RANK: 1 device-initiated comm, 0 NCCL, -1 auto
        int fold_comm = 1;         // device comm: pushes / halo wait inside the producers
        int band_rows = -1;        // SYM SpMV tile order: rows per band-plane (-1 auto, 0 off)
        int snake = -1;            // SYM SpMV: odd iterations visit the tiles last to first
        int comm_timeout_ms = 60000;   // device comm: spin limit before MINIFE_ECOMM
        int comm_fault_part = -1;  // fault injection (tests): this rank / part never signals
        int symm_nw = -1;          // SYM SpMV tile width: -1 auto (by N_x), 11 or 13
    } opt;
    bool devcomm_ready = false;                  // regions + peer tables built
    int cur_max_iters = 0;                       // max_iters of the solve being enqueued
    double last_asm_ms = 0.0, last_solve_ms = 0.0;   // device time, max over the parts
    std::vector<cudaGraphExec_t> gexec_parts;    // MULTI + device comm: one graph per device
    // kernel launch accounting: enq_kernels counts launch_* calls as they are enqueued (into a
    // capture or directly); g_kernels = kernels in the captured solve graph; kernel_launches =
    // kernels launched by this ctx so far (graph replays included)
    int64_t enq_kernels = 0, g_kernels = 0, kernel_launches = 0;
    // last solve
    int last_iters = 0;
    bool solved = false;
};

static void set_err(minife_ctx *c, const char *fmt, ...) {
    if (!c) return;
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
}

#define CUDA_TRY(ctx, call)                                                                   \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            set_err(ctx, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
            return e_ == cudaErrorMemoryAllocation ? MINIFE_ENOMEM : MINIFE_ECUDA;            \
        }                                                                                     \
    } while (0)

#define NCCL_TRY(ctx, call)                                                                   \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess) {                                                              \
            set_err(ctx, "%s: %s (%s:%d)", #call, nccl()->GetErrorString(r_), __FILE__,       \
                    __LINE__);                                                                \
            return MINIFE_ENCCL;                                                              \
        }                                                                                     \
    } while (0)

// one kernel of ours per launch_* wrapper (kernels.cu): counted for minife_info.kernel_launches
#define LAUNCH(ctx, call)                                                                     \
    do {                                                                                      \
        CUDA_TRY(ctx, call);                                                                  \
        ++(ctx)->enq_kernels;                                                                 \
    } while (0)

#define TRY(call)                                                                             \
    do {                                                                                      \
        int s_ = (call);                                                                      \
        if (s_ != MINIFE_OK) return s_;                                                       \
    } while (0)

static cudaStream_t stream_of(minife_ctx *c, Part &p) {
    if (c->user_stream && (c->mode == MINIFE_MODE_SINGLE || c->mode == MINIFE_MODE_RANK))
        return c->user_stream;
    return p.stream;
}

// all parts of a VIRTUAL ctx share part 0's stream (one device, one ordered queue)
static cudaStream_t launch_stream(minife_ctx *c, Part &p) {
    return c->mode == MINIFE_MODE_VIRTUAL ? c->parts[0].stream : stream_of(c, p);
}

template <class T>
static int dalloc(minife_ctx *c, Part &p, T **ptr, size_t n) {
    if (n == 0) n = 1;
    CUDA_TRY(c, cudaMalloc((void **)ptr, n * sizeof(T)));
    p.bytes += n * sizeof(T);
    return MINIFE_OK;
}

template <class T>
static void dfree(Part &p, T *&ptr, size_t n) {
    if (!ptr) return;
    cudaFree(ptr);
    ptr = nullptr;
    p.bytes -= (n ? n : 1) * sizeof(T);
}

// column vector (+32 doubles of padding: TMA tile copies round their size up to 16 B), zeroed
static int alloc_colvec(minife_ctx *c, Part &p, double **ptr) {
    const size_t n = (size_t)(p.ncols + 32);
    TRY(dalloc(c, p, ptr, n));
    // stream-ordered before every later kernel on the part's queue (the legacy-stream
    // cudaMemset is not ordered with the non-blocking ctx streams)
    CUDA_TRY(c, cudaMemsetAsync(*ptr, 0, n * sizeof(double), launch_stream(c, p)));
    return MINIFE_OK;
}

static void free_matrix(Part &p) {
    DevGuard g(p.dev);
    for (void **b : {(void **)&p.d_col, (void **)&p.d_seg, (void **)&p.d_mask, (void **)&p.d_val}) {
        if (*b) cudaFree(*b);
        *b = nullptr;
    }
    p.bytes -= p.matrix_bytes;
    p.matrix_bytes = 0;
    p.entries = 0;
}

static void free_part(Part &p) {
    DevGuard g(p.dev);
    free_matrix(p);
    void *bufs[] = {p.d_slice_off, p.d_row_len, p.d_width,   p.d_b,        p.d_x,
                    p.d_r,         p.d_p,       p.d_Ap,      p.d_xin,      p.d_yout,  p.d_p2,
                    p.d_acc,       p.d_st,      p.d_hist,    p.d_rr,       p.d_send_col,
                    p.d_recv_pos,  p.d_sendbuf, p.d_recvbuf, p.d_slice_row, p.d_slice_pos,
                    p.d_send_row,  p.d_push_nbr, p.d_push_dst, p.d_push_ptr, p.d_alpha,
                    p.d_comm,      p.d_comm_ptrs, p.d_nbr_rank, p.d_tile_order, p.d_rhalo,
                    p.d_rdst,      p.d_rhalo_ptr};
    for (void *q : p.ipc_opened) cudaIpcCloseMemHandle(q);
    for (void *b : bufs)
        if (b) cudaFree(b);
    for (double *b : p.d_pr)
        if (b) cudaFree(b);
    if (p.comm) nccl()->CommDestroy(p.comm);
    if (p.ev_push) cudaEventDestroy(p.ev_push);
    if (p.ev_fork) cudaEventDestroy(p.ev_fork);
    if (p.ev_t0) cudaEventDestroy(p.ev_t0);
    if (p.ev_t1) cudaEventDestroy(p.ev_t1);
    if (p.ev_join) cudaEventDestroy(p.ev_join);
    if (p.cstream) cudaStreamDestroy(p.cstream);
    if (p.stream) cudaStreamDestroy(p.stream);
}

static Geom geom_of(const minife_ctx *c, const Part &p) {
    Geom g{};
    g.nx = c->mesh.nx;
    g.ny = c->mesh.ny;
    g.nz = c->mesh.nz;
    for (int k = 0; k < 3; ++k) {
        g.own_lo[k] = p.plan.own_lo[k];
        g.own_n[k] = (int)p.plan.own_n[k];
        g.ext_lo[k] = p.plan.ext_lo[k];
        g.ext_n[k] = (int)p.plan.ext_n[k];
        g.off[k] = p.plan.off[k];
    }
    g.rows = p.rows;
    g.ncols = p.ncols;
    g.ident = p.ncols == p.rows;
    for (int k = 0; k < 2; ++k) {                 // ext_n >= 2 (a box has >= 2 nodes per axis)
        const unsigned __int128 two64 = (unsigned __int128)1 << 64;
        const uint64_t d = (uint64_t)std::max(2, g.ext_n[k]);
        g.ext_mag[k] = (uint64_t)((two64 + d - 1) / d);
    }
    return g;
}

// ----------------------------------------------------------------------------------------
// creation
// ----------------------------------------------------------------------------------------

static int alloc_hist(minife_ctx *c, Part &p, int cap) {
    DevGuard g(p.dev);
    dfree(p, p.d_hist, p.hist_cap);
    dfree(p, p.d_rr, p.hist_cap);
    dfree(p, p.d_alpha, p.hist_cap);
    TRY(dalloc(c, p, &p.d_hist, cap));
    TRY(dalloc(c, p, &p.d_rr, cap));
    TRY(dalloc(c, p, &p.d_alpha, cap));
    p.hist_cap = cap;
    return MINIFE_OK;
}

static int setup_part(minife_ctx *c, Part &p, int dev, const Plan &plan) {
    p.dev = dev;
    p.plan = plan;
    DevGuard g(dev);
    p.rows = plan.n_owned;
    p.ncols = plan.n_cols;
    p.nslices = (p.rows + 31) / 32;
    p.nnz = plan.local_nnz();
    p.nns = plan.local_nns();
    CUDA_TRY(c, cudaStreamCreateWithFlags(&p.stream, cudaStreamNonBlocking));
    CUDA_TRY(c, cudaEventCreate(&p.ev_t0));
    CUDA_TRY(c, cudaEventCreate(&p.ev_t1));
    TRY(dalloc(c, p, &p.d_slice_off, p.nslices + 1));
    TRY(dalloc(c, p, &p.d_row_len, p.nslices * 32));
    TRY(dalloc(c, p, &p.d_width, p.nslices));
    // vectors carry 32 doubles of padding: TMA tile copies round their size up to 16 B
    TRY(dalloc(c, p, &p.d_b, p.rows + 32));
    TRY(dalloc(c, p, &p.d_x, p.rows + 32));
    TRY(dalloc(c, p, &p.d_r, p.rows + 32));
    TRY(alloc_colvec(c, p, &p.d_p));
    TRY(dalloc(c, p, &p.d_Ap, p.rows + 32));
    TRY(dalloc(c, p, &p.d_acc, 4 * ACC_WORDS));
    TRY(dalloc(c, p, &p.d_st, 1));
    TRY(alloc_hist(c, p, 201));
    CUDA_TRY(c, cudaMemset(p.d_acc, 0, 4 * ACC_WORDS * sizeof(unsigned long long)));
    CUDA_TRY(c, cudaMemset(p.d_st, 0, sizeof(CgState)));
    // halo index lists, as extended columns
    std::vector<int32_t> send_col(plan.send_idx.size()), recv_pos(plan.n_ext);
    for (size_t i = 0; i < plan.send_idx.size(); ++i)
        send_col[i] = (int32_t)plan.row_to_col(plan.send_idx[i]);
    for (int64_t i = 0; i < plan.n_ext; ++i) recv_pos[i] = (int32_t)plan.ext_pos[i];
    std::vector<int32_t> send_row(plan.send_idx.begin(), plan.send_idx.end());
    TRY(dalloc(c, p, &p.d_send_row, send_row.size()));
    if (!send_row.empty())
        CUDA_TRY(c, cudaMemcpy(p.d_send_row, send_row.data(), 4 * send_row.size(),
                               cudaMemcpyHostToDevice));
    TRY(dalloc(c, p, &p.d_send_col, send_col.size()));
    TRY(dalloc(c, p, &p.d_sendbuf, send_col.size()));
    TRY(dalloc(c, p, &p.d_recv_pos, recv_pos.size()));
    TRY(dalloc(c, p, &p.d_recvbuf, recv_pos.size()));
    if (!send_col.empty())
        CUDA_TRY(c, cudaMemcpy(p.d_send_col, send_col.data(), 4 * send_col.size(),
                               cudaMemcpyHostToDevice));
    if (!recv_pos.empty())
        CUDA_TRY(c, cudaMemcpy(p.d_recv_pos, recv_pos.data(), 4 * recv_pos.size(),
                               cudaMemcpyHostToDevice));
    p.grid_upd = stream_grid(p.rows);
    // halo/interior overlap: interior-first slice storage order + a transport stream
    p.n_int = p.nslices;
    if (plan.n_ext > 0) {
        std::vector<int32_t> order, pos(p.nslices);
        p.n_int = plan.slice_order(order);
        for (int64_t q = 0; q < p.nslices; ++q) pos[order[q]] = (int32_t)q;
        TRY(dalloc(c, p, &p.d_slice_row, p.nslices));
        TRY(dalloc(c, p, &p.d_slice_pos, p.nslices));
        CUDA_TRY(c, cudaMemcpy(p.d_slice_row, order.data(), 4 * p.nslices, cudaMemcpyHostToDevice));
        CUDA_TRY(c, cudaMemcpy(p.d_slice_pos, pos.data(), 4 * p.nslices, cudaMemcpyHostToDevice));
        CUDA_TRY(c, cudaStreamCreateWithFlags(&p.cstream, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaEventCreateWithFlags(&p.ev_fork, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&p.ev_join, cudaEventDisableTiming));
    }
    return MINIFE_OK;
}

// Push tables (MINIFE_TRANSPORT_PUSH; MULTI ctxs with NCCL reductions): part p's slot j of
// its block for neighbor q lands in q's halo slot recv_off_q[p] + j, i.e. q's extended column
// ext_pos_q[...]; the store goes through q's p array as seen from p's device (the same pointer
// on one device, a peer pointer in MULTI ctxs: `remote_p` gives it).
template <class RemoteP>
static int build_push_tables(minife_ctx *c, Part &p, RemoteP remote_p) {
    const size_t ns = p.plan.send_idx.size();
    const size_t nn = p.plan.nbr.size();
    std::vector<uint8_t> nb(ns);
    std::vector<int32_t> dst(ns);
    std::vector<double *> ptr(nn, nullptr);
    for (size_t k = 0; k < nn; ++k) {
        const int qr = p.plan.nbr[k];
        Plan qown;
        const Plan *qp = nullptr;
        if (c->mode == MINIFE_MODE_RANK) {
            if (!build_plan(c->mesh, c->world, qr, qown)) return MINIFE_ESTATE;
            qp = &qown;
        } else {
            qp = &c->parts[qr].plan;
        }
        const Plan &q = *qp;
        auto it = std::lower_bound(q.nbr.begin(), q.nbr.end(), p.plan.rank);
        const size_t kq = (size_t)(it - q.nbr.begin());
        if (kq >= q.nbr.size() || q.nbr[kq] != p.plan.rank ||
            q.recv_cnt[kq] != p.plan.send_cnt[k] || k > 255) {
            set_err(c, "push plan mismatch between parts %d and %d", p.plan.rank, qr);
            return MINIFE_ESTATE;
        }
        for (int64_t j = 0; j < p.plan.send_cnt[k]; ++j) {
            nb[p.plan.send_off[k] + j] = (uint8_t)k;
            dst[p.plan.send_off[k] + j] = (int32_t)q.ext_pos[q.recv_off[kq] + j];
        }
        ptr[k] = remote_p(qr);
    }
    DevGuard g(p.dev);
    if (!p.d_push_nbr) {
        TRY(dalloc(c, p, &p.d_push_nbr, ns));
        TRY(dalloc(c, p, &p.d_push_dst, ns));
        TRY(dalloc(c, p, &p.d_push_ptr, ptr.size()));
    }
    if (ns) {
        CUDA_TRY(c, cudaMemcpy(p.d_push_nbr, nb.data(), ns, cudaMemcpyHostToDevice));
        CUDA_TRY(c, cudaMemcpy(p.d_push_dst, dst.data(), 4 * ns, cudaMemcpyHostToDevice));
    }
    if (!ptr.empty())
        CUDA_TRY(c, cudaMemcpy(p.d_push_ptr, ptr.data(), sizeof(double *) * ptr.size(),
                               cudaMemcpyHostToDevice));
    if (!p.ev_push) CUDA_TRY(c, cudaEventCreateWithFlags(&p.ev_push, cudaEventDisableTiming));
    CUDA_TRY(c, cudaDeviceSynchronize());     // legacy-stream copies above, see create_common
    return MINIFE_OK;
}

static int setup_push(minife_ctx *c) {
    for (auto &p : c->parts)
        TRY(build_push_tables(c, p, [c](int qr) { return c->parts[qr].d_p; }));
    c->push_ready = true;
    return MINIFE_OK;
}

// Halo by r (device comm): part p's send slot j for neighbour q lands in q's r-halo slot
// recv_off_q[p] + j; rhalo_of(q) = q's r-halo buffer as seen from p's device.
template <class RhaloOf>
static int build_rhalo_tables(minife_ctx *c, Part &p, RhaloOf rhalo_of) {
    const size_t ns = p.plan.send_idx.size(), nn = p.plan.nbr.size();
    std::vector<uint8_t> nb(ns);
    std::vector<int32_t> dst(ns);
    std::vector<double *> ptr(nn);
    for (size_t k = 0; k < nn; ++k) {
        const int qr = p.plan.nbr[k];
        Plan qown;
        if (!build_plan(c->mesh, c->world, qr, qown)) return MINIFE_ESTATE;
        auto it = std::lower_bound(qown.nbr.begin(), qown.nbr.end(), p.plan.rank);
        const size_t kq = (size_t)(it - qown.nbr.begin());
        if (kq >= qown.nbr.size() || qown.nbr[kq] != p.plan.rank ||
            qown.recv_cnt[kq] != p.plan.send_cnt[k] || k > 255) {
            set_err(c, "halo plan mismatch between parts %d and %d", p.plan.rank, qr);
            return MINIFE_ESTATE;
        }
        for (int64_t j = 0; j < p.plan.send_cnt[k]; ++j) {
            nb[p.plan.send_off[k] + j] = (uint8_t)k;
            dst[p.plan.send_off[k] + j] = (int32_t)(qown.recv_off[kq] + j);
        }
        ptr[k] = rhalo_of(qr);
    }
    DevGuard g(p.dev);
    if (!p.d_push_nbr) TRY(dalloc(c, p, &p.d_push_nbr, ns));
    if (!p.d_rdst) TRY(dalloc(c, p, &p.d_rdst, ns));
    if (!p.d_rhalo_ptr) TRY(dalloc(c, p, &p.d_rhalo_ptr, nn));
    if (ns) {
        CUDA_TRY(c, cudaMemcpy(p.d_push_nbr, nb.data(), ns, cudaMemcpyHostToDevice));
        CUDA_TRY(c, cudaMemcpy(p.d_rdst, dst.data(), 4 * ns, cudaMemcpyHostToDevice));
    }
    if (nn)
        CUDA_TRY(c, cudaMemcpy(p.d_rhalo_ptr, ptr.data(), sizeof(double *) * nn,
                               cudaMemcpyHostToDevice));
    CUDA_TRY(c, cudaDeviceSynchronize());
    return MINIFE_OK;
}

// Device comm regions (DevComm, kernels.h) of every part of this ctx, zeroed, plus the
// neighbor-rank lists; `region_of(p, r)` = rank r's region as seen from part p's device.
template <class RegionOf>
static int setup_comm_tables(minife_ctx *c, RegionOf region_of) {
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        std::vector<unsigned long long *> regs(c->world);
        for (int r = 0; r < c->world; ++r) regs[r] = region_of(p, r);
        if (!p.d_comm_ptrs) TRY(dalloc(c, p, &p.d_comm_ptrs, c->world));
        CUDA_TRY(c, cudaMemcpy(p.d_comm_ptrs, regs.data(), sizeof(void *) * c->world,
                               cudaMemcpyHostToDevice));
        std::vector<int32_t> nbr(p.plan.nbr.begin(), p.plan.nbr.end());
        if (!p.d_nbr_rank) TRY(dalloc(c, p, &p.d_nbr_rank, nbr.size()));
        if (!nbr.empty())
            CUDA_TRY(c, cudaMemcpy(p.d_nbr_rank, nbr.data(), 4 * nbr.size(),
                                   cudaMemcpyHostToDevice));
        CUDA_TRY(c, cudaDeviceSynchronize());
    }
    return MINIFE_OK;
}

static int alloc_comm_regions(minife_ctx *c) {
    const int64_t words = comm_words(c->world);
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        if (!p.d_rhalo) {
            TRY(dalloc(c, p, &p.d_rhalo, (size_t)p.plan.n_ext));
            CUDA_TRY(c, cudaMemset(p.d_rhalo, 0, 8 * (size_t)std::max<int64_t>(1, p.plan.n_ext)));
        }
        if (!p.d_comm) TRY(dalloc(c, p, &p.d_comm, words));
        CUDA_TRY(c, cudaMemset(p.d_comm, 0, 8 * (size_t)words));
        CUDA_TRY(c, cudaDeviceSynchronize());
    }
    return MINIFE_OK;
}

// VIRTUAL and MULTI (peer access enabled): every region is addressable from every device
static int setup_devcomm_local(minife_ctx *c) {
    TRY(alloc_comm_regions(c));
    TRY(setup_comm_tables(c, [c](Part &, int r) { return c->parts[r].d_comm; }));
    for (auto &p : c->parts)
        TRY(build_rhalo_tables(c, p, [c](int qr) { return c->parts[qr].d_rhalo; }));
    c->devcomm_ready = true;
    return MINIFE_OK;
}

// RANK ctxs (one process per GPU, torchrun): the comm region and the r-halo buffer of every
// rank are exported as CUDA-IPC handles and exchanged once with an NCCL all-gather; each rank
// maps every other rank's region and its neighbours' r-halo buffers.  The ranks then agree
// (NCCL MIN all-reduce) whether every mapping succeeded: if any rank failed (no P2P between
// some pair, IPC unavailable), all of them keep the NCCL transport.  Collective over the ranks.
struct IpcRecord {
    cudaIpcMemHandle_t comm, rhalo;
    int32_t dev, ok;
};

static int setup_devcomm_ipc(minife_ctx *c) {
    Part &p = c->parts[0];
    DevGuard g(p.dev);
    TRY(alloc_comm_regions(c));
    const int W = c->world, R = c->rank;
    IpcRecord mine{};
    mine.dev = p.dev;
    mine.ok = cudaIpcGetMemHandle(&mine.comm, p.d_comm) == cudaSuccess &&
              cudaIpcGetMemHandle(&mine.rhalo, p.d_rhalo) == cudaSuccess;
    cudaGetLastError();
    std::vector<IpcRecord> all(W);
    IpcRecord *d_all = nullptr;
    int32_t *d_ok = nullptr;
    CUDA_TRY(c, cudaMalloc((void **)&d_all, sizeof(IpcRecord) * W));
    CUDA_TRY(c, cudaMalloc((void **)&d_ok, sizeof(int32_t)));
    int st = MINIFE_OK;
    cudaError_t e = cudaMemcpyAsync(d_all + R, &mine, sizeof mine, cudaMemcpyHostToDevice, p.stream);
    ncclResult_t nr = ncclSuccess;
    if (e == cudaSuccess)
        nr = nccl()->AllGather(d_all + R, d_all, sizeof(IpcRecord), ncclUint8, p.comm, p.stream);
    if (e == cudaSuccess && nr == ncclSuccess)
        e = cudaMemcpyAsync(all.data(), d_all, sizeof(IpcRecord) * W, cudaMemcpyDeviceToHost,
                            p.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p.stream);
    if (e != cudaSuccess || nr != ncclSuccess) {
        set_err(c, "IPC handle exchange: %s / %s", cudaGetErrorString(e),
                nccl()->GetErrorString(nr));
        st = e != cudaSuccess ? MINIFE_ECUDA : MINIFE_ENCCL;
    }
    // map every other rank's region, and the neighbours' r-halo buffers
    std::vector<unsigned long long *> regions(W, nullptr);
    std::vector<double *> rhalo(W, nullptr);
    int32_t ok = st == MINIFE_OK ? 1 : 0;
    for (int r = 0; r < W && ok; ++r) {
        if (!all[r].ok) ok = 0;
        if (r == R) {
            regions[r] = p.d_comm;
            rhalo[r] = p.d_rhalo;
            continue;
        }
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, p.dev, all[r].dev) != cudaSuccess || !can) ok = 0;
        void *q = nullptr;
        if (ok && cudaIpcOpenMemHandle(&q, all[r].comm, cudaIpcMemLazyEnablePeerAccess) ==
                      cudaSuccess) {
            p.ipc_opened.push_back(q);
            regions[r] = (unsigned long long *)q;
        } else {
            ok = 0;
        }
        if (ok && std::binary_search(p.plan.nbr.begin(), p.plan.nbr.end(), r)) {
            if (cudaIpcOpenMemHandle(&q, all[r].rhalo, cudaIpcMemLazyEnablePeerAccess) ==
                cudaSuccess) {
                p.ipc_opened.push_back(q);
                rhalo[r] = (double *)q;
            } else {
                ok = 0;
            }
        }
        cudaGetLastError();
    }
    // every rank must take the same transport
    if (st == MINIFE_OK) {
        e = cudaMemcpyAsync(d_ok, &ok, sizeof ok, cudaMemcpyHostToDevice, p.stream);
        if (e == cudaSuccess)
            nr = nccl()->AllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, p.comm, p.stream);
        if (e == cudaSuccess && nr == ncclSuccess)
            e = cudaMemcpyAsync(&ok, d_ok, sizeof ok, cudaMemcpyDeviceToHost, p.stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(p.stream);
        if (e != cudaSuccess || nr != ncclSuccess) {
            set_err(c, "transport agreement: %s / %s", cudaGetErrorString(e),
                    nccl()->GetErrorString(nr));
            st = e != cudaSuccess ? MINIFE_ECUDA : MINIFE_ENCCL;
        }
    }
    cudaFree(d_all);
    cudaFree(d_ok);
    if (st != MINIFE_OK) return st;
    if (!ok) {                                   // NCCL transport on every rank
        for (void *q : p.ipc_opened) cudaIpcCloseMemHandle(q);
        p.ipc_opened.clear();
        cudaGetLastError();
        return MINIFE_OK;
    }
    TRY(setup_comm_tables(c, [&regions](Part &, int r) { return regions[r]; }));
    if (W > 1) TRY(build_rhalo_tables(c, p, [&rhalo](int qr) { return rhalo[qr]; }));
    c->devcomm_ready = true;
    return MINIFE_OK;
}

// MULTI ctxs: peer access between every device pair -> push transport over NVLink
static bool enable_peers(minife_ctx *c) {
    for (auto &a : c->parts)
        for (auto &b : c->parts) {
            if (a.dev == b.dev) continue;
            int ok = 0;
            if (cudaDeviceCanAccessPeer(&ok, a.dev, b.dev) != cudaSuccess || !ok) return false;
            DevGuard g(a.dev);
            const cudaError_t e = cudaDeviceEnablePeerAccess(b.dev, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return false;
            cudaGetLastError();
        }
    return true;
}

// Device-initiated comm in use for the next solve: VIRTUAL with MINIFE_TRANSPORT_DEVICE; MULTI
// and RANK when the regions are mapped (peer access / CUDA IPC) unless option device_comm = 0
// (RANK at world 1 only when forced with device_comm = 1: it exercises the same kernels).
static bool devcomm(const minife_ctx *c) {
    if (!c->devcomm_ready) return false;
    if (c->mode == MINIFE_MODE_VIRTUAL) return c->world > 1 && c->transport == MINIFE_TRANSPORT_DEVICE;
    if (c->world == 1) return c->mode == MINIFE_MODE_RANK && c->opt.device_comm == 1;
    return c->opt.device_comm != 0;
}

// Device comm with the pushes / halo wait folded into the producing kernels' last CTAs (the
// SYM path; SEG/CRS keep the separate k_acc_push launches).  Option
// "fold_comm" = 0 keeps the separate launches everywhere (tests compare both).
static bool fold_comm(const minife_ctx *c) {
    return devcomm(c) && c->fmt == MINIFE_FMT_SYM && c->opt.fold_comm != 0;
}

static bool push_mode(const minife_ctx *c) {
    if (devcomm(c)) return false;                // device comm: halo by r (enqueue_solve_dev)
    return c->world > 1 && c->push_ready &&
           (c->mode == MINIFE_MODE_MULTI ||
            (c->mode == MINIFE_MODE_VIRTUAL && c->transport == MINIFE_TRANSPORT_PUSH));
}

static UpdArgs upd_args(const minife_ctx *c, Part &p, int which_in);

// MULTI with NCCL reductions and the push transport: each part's compute stream waits for
// its neighbors' push kernels
static int push_wait(minife_ctx *c) {
    if (c->mode != MINIFE_MODE_MULTI) return MINIFE_OK;
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        for (int q : p.plan.nbr) CUDA_TRY(c, cudaStreamWaitEvent(p.stream, c->parts[q].ev_push, 0));
    }
    return MINIFE_OK;
}

// Device time of an operation enqueued on every part: events on each part's queue before
// and after; the duration is the max over the parts (CUDA events, not host clocks).
// (assembly runs on every part's own queue, the solve on launch_stream)
static int mark_parts(minife_ctx *c, bool end, bool assembly = false) {
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        cudaStream_t s = assembly ? stream_of(c, p) : launch_stream(c, p);
        CUDA_TRY(c, cudaEventRecord(end ? p.ev_t1 : p.ev_t0, s));
    }
    return MINIFE_OK;
}
static int elapsed_parts(minife_ctx *c, double *ms_out, double Part::*per_part) {
    double mx = 0.0;
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        CUDA_TRY(c, cudaEventSynchronize(p.ev_t1));
        float ms = 0.f;
        CUDA_TRY(c, cudaEventElapsedTime(&ms, p.ev_t0, p.ev_t1));
        p.*per_part = ms;
        mx = std::max(mx, (double)ms);
    }
    *ms_out = mx;
    return MINIFE_OK;
}

static int validate_mesh(int nx, int ny, int nz) {
    if (nx < 1 || ny < 1 || nz < 1) return MINIFE_EINVAL;
    return MINIFE_OK;
}

static int create_common(minife_ctx *c, int nx, int ny, int nz, int nparts,
                         const std::vector<int> &devs, int rank_only) {
    c->mesh = Mesh{nx, ny, nz};
    std::vector<Box> boxes;
    if (!rcb(c->mesh, c->world, boxes)) {
        set_err(c, "RCB: %d ranks do not fit a %dx%dx%d element mesh (S:65)", c->world, nx, ny,
                nz);
        return MINIFE_EINVAL;
    }
    c->parts.resize(nparts);
    for (int q = 0; q < nparts; ++q) {
        const int r = rank_only >= 0 ? rank_only : q;
        Plan plan;
        if (!build_plan(c->mesh, c->world, r, plan)) {
            set_err(c, "plan construction failed for rank %d", r);
            return MINIFE_EINVAL;
        }
        if (plan.n_cols >= ((int64_t)1 << 31) - 64) {
            set_err(c, "part %d has %lld columns: int32 local indices overflow", r,
                    (long long)plan.n_cols);
            return MINIFE_EINVAL;
        }
        TRY(setup_part(c, c->parts[q], devs[q], plan));
    }
    // default format: SYM (B200, 300^3: SYM SpMV 0.88 ms vs SEG 1.07 ms; with a halo the
    // halo nodes are stored as ghost rows, profiles/r01/session2)
    c->fmt = MINIFE_FMT_SYM;
    // the setup copies/memsets above ran on the legacy stream: complete them before any
    // kernel on the (non-blocking) ctx streams can touch those buffers
    for (auto &p : c->parts) {
        DevGuard gp(p.dev);
        CUDA_TRY(c, cudaDeviceSynchronize());
    }
    DevGuard g(c->parts[0].dev);
    CUDA_TRY(c, cudaEventCreate(&c->ev0));
    CUDA_TRY(c, cudaEventCreate(&c->ev1));
    return MINIFE_OK;
}

extern "C" int minife_create(int nx, int ny, int nz, int ngpu, minife_ctx **out) {
    if (!out || validate_mesh(nx, ny, nz) != MINIFE_OK || ngpu < 1) return MINIFE_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return MINIFE_ENODEV;
    if (ngpu > ndev) return MINIFE_ENODEV;
    minife_ctx *c = new minife_ctx();
    c->mode = ngpu == 1 ? MINIFE_MODE_SINGLE : MINIFE_MODE_MULTI;
    c->world = ngpu;
    std::vector<int> devs(ngpu);
    for (int q = 0; q < ngpu; ++q) devs[q] = q;
    int st = create_common(c, nx, ny, nz, ngpu, devs, -1);
    if (st == MINIFE_OK && ngpu > 1 && !nccl()) {
        set_err(c, "NCCL could not be loaded (set MINIFE_NCCL_LIB)");
        st = MINIFE_ENCCL;
    }
    if (st == MINIFE_OK && ngpu > 1) {
        std::vector<ncclComm_t> comms(ngpu);
        ncclResult_t r = nccl()->CommInitAll(comms.data(), ngpu, devs.data());
        if (r != ncclSuccess) {
            set_err(c, "ncclCommInitAll: %s", nccl()->GetErrorString(r));
            st = MINIFE_ENCCL;
        } else {
            for (int q = 0; q < ngpu; ++q) c->parts[q].comm = comms[q];
        }
    }
    // peer access between every device pair: halo push over NVLink and device-initiated
    // reductions (comm regions addressed through peer pointers); otherwise NCCL throughout
    if (st == MINIFE_OK && ngpu > 1 && enable_peers(c)) {
        st = setup_push(c);
        if (st == MINIFE_OK) st = setup_devcomm_local(c);
    }
    if (st != MINIFE_OK) {
        minife_destroy(c);
        return st;
    }
    *out = c;
    return MINIFE_OK;
}

extern "C" int minife_create_virtual(int nx, int ny, int nz, int nparts, minife_ctx **out) {
    if (!out || validate_mesh(nx, ny, nz) != MINIFE_OK || nparts < 1 || nparts > 64)
        return MINIFE_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return MINIFE_ENODEV;
    minife_ctx *c = new minife_ctx();
    c->mode = MINIFE_MODE_VIRTUAL;
    c->world = nparts;
    std::vector<int> devs(nparts, 0);
    int st = create_common(c, nx, ny, nz, nparts, devs, -1);
    if (st == MINIFE_OK && nparts > 1) st = setup_push(c);
    if (st == MINIFE_OK && nparts > 1) st = setup_devcomm_local(c);
    if (st != MINIFE_OK) {
        minife_destroy(c);
        return st;
    }
    *out = c;
    return MINIFE_OK;
}

extern "C" int minife_nccl_unique_id(void *uid128) {
    if (!uid128) return MINIFE_EINVAL;
    ncclUniqueId id;
    if (!nccl() || nccl()->GetUniqueId(&id) != ncclSuccess) return MINIFE_ENCCL;
    memcpy(uid128, &id, sizeof id);
    return MINIFE_OK;
}

extern "C" int minife_create_rank(int nx, int ny, int nz, int rank, int world, int device,
                                  const void *uid128, minife_ctx **out) {
    if (!out || !uid128 || validate_mesh(nx, ny, nz) != MINIFE_OK || world < 1 || rank < 0 ||
        rank >= world || device < 0)
        return MINIFE_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1 || device >= ndev)
        return MINIFE_ENODEV;
    minife_ctx *c = new minife_ctx();
    c->mode = MINIFE_MODE_RANK;
    c->world = world;
    c->rank = rank;
    std::vector<int> devs(1, device);
    int st = create_common(c, nx, ny, nz, 1, devs, rank);
    if (st == MINIFE_OK && !nccl()) {
        set_err(c, "NCCL could not be loaded (set MINIFE_NCCL_LIB)");
        st = MINIFE_ENCCL;
    }
    if (st == MINIFE_OK) {
        DevGuard g(device);
        ncclUniqueId id;
        memcpy(&id, uid128, sizeof id);
        ncclResult_t r = nccl()->CommInitRank(&c->parts[0].comm, world, id, rank);
        if (r != ncclSuccess) {
            set_err(c, "ncclCommInitRank: %s", nccl()->GetErrorString(r));
            st = MINIFE_ENCCL;
        }
    }
    if (st == MINIFE_OK) st = setup_devcomm_ipc(c);
    if (st != MINIFE_OK) {
        minife_destroy(c);
        return st;
    }
    *out = c;
    return MINIFE_OK;
}

static void drop_graph(minife_ctx *c) {
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    c->gexec = nullptr;
    for (auto ex : c->gexec_parts) cudaGraphExecDestroy(ex);
    c->gexec_parts.clear();
    c->g_iters = -1;
}

extern "C" void minife_destroy(minife_ctx *c) {
    if (!c) return;
    drop_graph(c);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (!c->parts.empty()) {
        DevGuard g(c->parts[0].dev);
        for (cudaEvent_t e : c->tw_ev) cudaEventDestroy(e);
    }
    for (auto &p : c->parts) free_part(p);
    delete c;
}

extern "C" int minife_set_stream(minife_ctx *c, void *stream) {
    if (!c) return MINIFE_EINVAL;
    if (c->mode != MINIFE_MODE_SINGLE && c->mode != MINIFE_MODE_RANK) return MINIFE_ESTATE;
    c->user_stream = (cudaStream_t)stream;
    return MINIFE_OK;
}

extern "C" int minife_set_option(minife_ctx *c, const char *name, int64_t value) {
    if (!c || !name) return MINIFE_EINVAL;
    struct {
        const char *name;
        int *field;
        int lo, hi;
    } table[] = {
        {"x_defer", &c->opt.x_defer, -1, XDEF_MAX},
        {"small_solver", &c->opt.small_solver, -1, 2},
        {"graph", &c->opt.graph, 0, 1},
        {"val_evict_first", &c->opt.val_evict_first, -1, 1},
        {"x_prefetch", &c->opt.x_prefetch, -1, 1},
        {"sym_kernel", &c->opt.sym_kernel, 0, 1},
        {"spmv_impl", &c->opt.spmv_impl, -1, 1},
        {"x_late", &c->opt.x_late, 0, 1},
        {"cluster_dd", &c->opt.cluster_dd, 0, 1},
        {"device_comm", &c->opt.device_comm, -1, 1},
        {"fold_comm", &c->opt.fold_comm, 0, 1},
        {"band_rows", &c->opt.band_rows, -1, 1 << 30},
        {"snake", &c->opt.snake, -1, 1},
        {"comm_timeout_ms", &c->opt.comm_timeout_ms, 1, 3600000},
        {"comm_fault_part", &c->opt.comm_fault_part, -1, 1 << 20},
        {"symm_nw", &c->opt.symm_nw, -1, SYMM_NW},
    };
    for (auto &t : table) {
        if (strcmp(t.name, name) != 0) continue;
        if (value < t.lo || value > t.hi ||
            (t.field == &c->opt.symm_nw && value != -1 && value != SYMM_NW &&
             value != SYMM_NW_WIDE)) {
            set_err(c, "option %s: value %lld outside [%d, %d]", name, (long long)value, t.lo, t.hi);
            return MINIFE_EINVAL;
        }
        if (*t.field != (int)value) {
            *t.field = (int)value;
            drop_graph(c);
        }
        return MINIFE_OK;
    }
    set_err(c, "unknown option %s", name);
    return MINIFE_EINVAL;
}

extern "C" int minife_set_transport(minife_ctx *c, int transport) {
    if (!c || (transport != MINIFE_TRANSPORT_DIRECT && transport != MINIFE_TRANSPORT_WIRE &&
               transport != MINIFE_TRANSPORT_PUSH && transport != MINIFE_TRANSPORT_DEVICE))
        return MINIFE_EINVAL;
    if (c->mode != MINIFE_MODE_VIRTUAL) return MINIFE_ESTATE;
    if (transport != c->transport) {
        c->transport = transport;
        drop_graph(c);
    }
    return MINIFE_OK;
}

extern "C" int minife_set_scheme(minife_ctx *c, int scheme) {
    if (!c || (scheme != MINIFE_SCHEME_3K && scheme != MINIFE_SCHEME_FUSED)) return MINIFE_EINVAL;
    if (scheme != c->scheme) {
        c->scheme = scheme;
        drop_graph(c);
    }
    return MINIFE_OK;
}

extern "C" int minife_set_format(minife_ctx *c, int format) {
    if (!c || (format != MINIFE_FMT_CRS && format != MINIFE_FMT_SEG && format != MINIFE_FMT_SYM))
        return MINIFE_EINVAL;

    if (format != c->fmt) {
        c->fmt = format;
        c->assembled = false;
        c->solved = false;
        drop_graph(c);
        for (auto &p : c->parts) free_matrix(p);
    }
    return MINIFE_OK;
}

extern "C" const char *minife_strerror(int s) {
    switch (s) {
    case MINIFE_OK: return "ok";
    case MINIFE_EINVAL: return "invalid argument";
    case MINIFE_ESTATE: return "invalid state for this call";
    case MINIFE_ECUDA: return "CUDA error";
    case MINIFE_ENCCL: return "NCCL error";
    case MINIFE_ENOMEM: return "out of memory";
    case MINIFE_ENOTSPD: return "matrix not SPD (pAp <= 0 with rr != 0)";
    case MINIFE_EDIVERGED: return "CG diverged (non-finite value)";
    case MINIFE_ENODEV: return "no (or not enough) CUDA devices";
    case MINIFE_ECOMM: return "device-initiated comm: a peer did not signal in time";
    default: return "unknown status";
    }
}

extern "C" const char *minife_last_error(const minife_ctx *c) { return c ? c->err.c_str() : ""; }

extern "C" int minife_bandwidth_probe(int device, int64_t bytes, int reps, double *read_gbs,
                                      double *copy_gbs) {
    if (bytes < (1 << 20) || reps < 1 || !read_gbs || !copy_gbs) return MINIFE_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return MINIFE_ENODEV;
    DevGuard g(device);
    cudaError_t e = probe_bandwidth(bytes, reps, read_gbs, copy_gbs);
    if (e == cudaErrorMemoryAllocation) return MINIFE_ENOMEM;
    return e == cudaSuccess ? MINIFE_OK : MINIFE_ECUDA;
}

extern "C" int minife_dot(int device, int64_t n, const double *u, const double *v, double *out) {
    if (!out || n < 0 || n >= ((int64_t)1 << 29) || (n > 0 && (!u || !v))) return MINIFE_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return MINIFE_ENODEV;
    DevGuard g(device);
    static_assert(MINIFE_ACC_WORDS == ACC_WORDS, "accumulator layout");
    const size_t acc_b = ACC_WORDS * sizeof(unsigned long long);
    const size_t vec_b = (size_t)n * sizeof(double);
    unsigned char *buf = nullptr;
    if (cudaMalloc(&buf, acc_b + 64 + 2 * vec_b) != cudaSuccess) return MINIFE_ENOMEM;
    auto *acc = reinterpret_cast<unsigned long long *>(buf);
    auto *res = reinterpret_cast<double *>(buf + acc_b);
    auto *du = reinterpret_cast<double *>(buf + acc_b + 64);
    double *dv = du + n;
    cudaError_t e = cudaMemset(acc, 0, acc_b);
    if (e == cudaSuccess && n > 0) e = cudaMemcpy(du, u, vec_b, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && n > 0) e = cudaMemcpy(dv, v, vec_b, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_dot(du, dv, n, acc, 0);
    if (e == cudaSuccess) e = launch_acc_round(acc, res, 0);
    if (e == cudaSuccess) e = cudaMemcpy(out, res, sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(buf);
    return e == cudaSuccess ? MINIFE_OK : MINIFE_ECUDA;
}

extern "C" int minife_exact_round(int device, const int64_t *words, double *out) {
    if (!words || !out) return MINIFE_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return MINIFE_ENODEV;
    DevGuard g(device);
    const size_t acc_b = ACC_WORDS * sizeof(unsigned long long);
    unsigned char *buf = nullptr;
    if (cudaMalloc(&buf, acc_b + 64) != cudaSuccess) return MINIFE_ENOMEM;
    auto *acc = reinterpret_cast<unsigned long long *>(buf);
    auto *res = reinterpret_cast<double *>(buf + acc_b);
    cudaError_t e = cudaMemcpy(acc, words, acc_b, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_acc_round(acc, res, 0);
    if (e == cudaSuccess) e = cudaMemcpy(out, res, sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(buf);
    return e == cudaSuccess ? MINIFE_OK : MINIFE_ECUDA;
}

namespace minife {
extern double g_l2_read_gbs;
extern double g_write_gbs;
}
extern "C" double minife_probe_l2_read_gbs(void) { return minife::g_l2_read_gbs; }
extern "C" double minife_probe_write_gbs(void) { return minife::g_write_gbs; }
extern "C" const char *minife_version(void) { return MINIFE_VERSION; }

// ----------------------------------------------------------------------------------------
// assembly (a0.2 - a0.5)
// ----------------------------------------------------------------------------------------

// SYM storage: by extended column (ghost rows for the halo nodes) -- slices over ncols
static int64_t sym_slices(const Part &p) { return (p.ncols + 31) / 32; }

static Matrix matrix_of(const minife_ctx *c, const Part &p) {
    Matrix m{};
    m.fmt = c->fmt;
    m.rows = p.rows;
    m.nslices = p.nslices;
    if (c->fmt == MINIFE_FMT_SYM) {
        m.ext = p.ncols != p.rows;
        m.rows = p.ncols;
        m.nslices = sym_slices(p);
    }
    m.val = p.d_val;
    m.slice_off = p.d_slice_off;
    m.row_len = p.d_row_len;
    m.col = p.d_col;
    m.seg = p.d_seg;
    m.mask = p.d_mask;
    if (c->fmt == MINIFE_FMT_SEG) {          // interior-first slice order (null: identity)
        m.slice_row = p.d_slice_row;
        m.slice_pos = p.d_slice_pos;
    }
    return m;
}

// SYM SpMV tile order: a row's plane-back mirrors (its dz = -1 runs) come from
// the row one plane earlier, which the SpMV streamed ~one plane of tiles ago; past ~14 MB of
// matrix per plane (400^3: 24 MB) part of them is evicted from L2 before it is read again
// (400^3 read 8-15 % above the algorithmic bytes).  Planes of more than BAND_MIN_PLANE rows
// are visited band-major: y-bands of B = band_rows / N0 lines, each swept plane by plane, so
// the plane-back rows are B lines back instead of a plane.  B200, interleaved A/B
// (profiles/r02/ab): 400^3 band_rows 65536 SpMV 1.82 vs 1.89 ms, DRAM reads 10.37 vs
// 10.8-11.6 GB (algorithmic 10.0), 49152 / 98304 / 131072 worse; 300^3 (90.6K-row planes)
// is 10 % SLOWER banded at any band size with the same DRAM bytes, so it stays natural.
static constexpr int64_t BAND_ROWS_AUTO = 65536, BAND_MIN_PLANE = 122880;
static int build_tile_order(minife_ctx *c, Part &p) {
    DevGuard g(p.dev);
    // a captured solve graph holds the order's device pointer: the buffer is reused when the
    // order keeps its size (re-assembly), and any other change drops the graph
    auto drop_order = [&]() {
        if (!p.d_tile_order) return;
        dfree(p, p.d_tile_order, (size_t)p.tile_order_n);
        p.tile_order_n = 0;
        drop_graph(c);
    };
    const int64_t N0 = p.plan.ext_n[0], N1 = p.plan.ext_n[1];
    // the tile width the SpMV runs with: the order is in its tiles, so both change together
    const int nw = c->opt.symm_nw > 0 ? c->opt.symm_nw : symm_nw_auto(N0);
    if (nw != p.symm_nw) {
        p.symm_nw = nw;
        drop_graph(c);
    }
    if (c->fmt != MINIFE_FMT_SYM) {
        drop_order();
        return MINIFE_OK;
    }
    const int64_t P = N0 * N1;
    const int64_t target = c->opt.band_rows < 0 ? BAND_ROWS_AUTO : c->opt.band_rows;
    if (target == 0 || (c->opt.band_rows < 0 && P <= BAND_MIN_PLANE) || P <= target) {
        drop_order();
        return MINIFE_OK;
    }
    const int64_t B = std::max<int64_t>(8, target / N0);               // lines per band
    const int64_t nslices = (p.ncols + 31) / 32;
    const int64_t ntiles = (nslices + nw - 1) / nw;
    std::vector<std::pair<int64_t, int32_t>> key(ntiles);
    for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t r = t * nw * 32;
        const int64_t ey = (r / N0) % N1, ez = r / P;
        key[t] = {(ey / B) * (int64_t)1e12 + ez * (int64_t)1e6 + 0, (int32_t)t};
    }
    std::stable_sort(key.begin(), key.end(),
                     [](const std::pair<int64_t, int32_t> &x, const std::pair<int64_t, int32_t> &y) {
                         return x.first < y.first;
                     });
    std::vector<int32_t> order(ntiles);
    for (int64_t t = 0; t < ntiles; ++t) order[t] = key[t].second;
    if (p.d_tile_order && p.tile_order_n != ntiles) drop_order();
    if (!p.d_tile_order) {
        TRY(dalloc(c, p, &p.d_tile_order, (size_t)ntiles));
        p.tile_order_n = ntiles;
        drop_graph(c);
    }
    CUDA_TRY(c, cudaMemcpy(p.d_tile_order, order.data(), 4 * (size_t)ntiles, cudaMemcpyHostToDevice));
    return MINIFE_OK;
}

extern "C" int minife_assemble(minife_ctx *c) {
    NvtxRange nvtx_("minife_assemble");
    if (!c) return MINIFE_EINVAL;
    // CRS sizes its arrays from a device pass read back to the host: its time is host-split
    const bool timed = c->fmt != MINIFE_FMT_CRS;
    for (auto &p : c->parts) TRY(build_tile_order(c, p));   // (legacy-stream copy: before the
    for (auto &p : c->parts) {                               //  kernels on the part streams)
        DevGuard g(p.dev);
        CUDA_TRY(c, cudaDeviceSynchronize());
    }
    if (timed) TRY(mark_parts(c, false, true));
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        cudaStream_t s = stream_of(c, p);
        const Geom geo = geom_of(c, p);
        AsmArgs a{};
        a.g = geo;
        a.fmt = c->fmt;
        if (c->fmt == MINIFE_FMT_CRS) {
            // slice widths on the device, offsets by a host prefix sum (8 B per 32 rows)
            LAUNCH(c, launch_rowlen_widths(geo, p.d_row_len, p.d_width, p.nslices, s));
            std::vector<uint8_t> w(p.nslices);
            CUDA_TRY(c, cudaMemcpyAsync(w.data(), p.d_width, p.nslices, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(c, cudaStreamSynchronize(s));
            p.h_slice_off.assign(p.nslices + 1, 0);
            for (int64_t i = 0; i < p.nslices; ++i)
                p.h_slice_off[i + 1] = p.h_slice_off[i] + 32 * (int64_t)w[i];
            const int64_t entries = p.h_slice_off[p.nslices];
            if (entries != p.entries || !p.d_col) {
                free_matrix(p);
                TRY(dalloc(c, p, &p.d_col, entries));
                TRY(dalloc(c, p, &p.d_val, entries));
                p.matrix_bytes = 12 * (size_t)entries;
                p.entries = entries;
            }
            CUDA_TRY(c, cudaMemcpyAsync(p.d_slice_off, p.h_slice_off.data(), 8 * (p.nslices + 1),
                                        cudaMemcpyHostToDevice, s));
            CUDA_TRY(c, cudaStreamSynchronize(s));
        } else {
            // SEG: 27 value slots per row; SYM: the 14 upper slots, stored for every node of
            // the extended box (ghost rows for the halo nodes; = the rows with one part)
            const bool sym = c->fmt == MINIFE_FMT_SYM;
            const int64_t ns = sym ? sym_slices(p) : p.nslices;
            const int64_t entries = (sym ? 14 : 27) * 32 * ns;
            if (!p.d_seg || entries != p.entries) {
                free_matrix(p);
                TRY(dalloc(c, p, &p.d_val, entries));
                const size_t vbytes = 8 * (size_t)entries;
                TRY(dalloc(c, p, &p.d_seg, 9 * 32 * ns));
                TRY(dalloc(c, p, &p.d_mask, 32 * ns));           // padded: whole-slice copies
                p.matrix_bytes = vbytes + 4 * (size_t)(9 * 32 * ns) + 4 * (size_t)(32 * ns);
                p.entries = entries;
            }
        }
        a.slice_off = p.d_slice_off;
        a.row_len = p.d_row_len;
        a.col = p.d_col;
        a.seg = p.d_seg;
        a.mask = p.d_mask;
        a.val = p.d_val;
        a.b = p.d_b;
        a.slice_pos = c->fmt == MINIFE_FMT_SEG ? p.d_slice_pos : nullptr;
        LAUNCH(c, launch_assemble(a, s));
        p.grid_spmv = spmv_grid(p.nslices, c->fmt);
    }
    if (timed) TRY(mark_parts(c, true, true));
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        CUDA_TRY(c, cudaStreamSynchronize(stream_of(c, p)));
    }
    c->last_asm_ms = 0.0;
    if (timed) TRY(elapsed_parts(c, &c->last_asm_ms, &Part::t_asm_ms));
    c->assembled = true;
    c->solved = false;
    return MINIFE_OK;
}

// ----------------------------------------------------------------------------------------
// transports: halo exchange (a1) and accumulator all-reduce (a3/a5)
// ----------------------------------------------------------------------------------------

// Push the halo of p (mode 0: current p; mode 1: p_(k+1) ahead of K7) from every part, then
// (MULTI) make every part's compute stream wait for its neighbors' pushes.  With mode 1 the
// waits are placed by the caller after K7 (wait_now = false).
static int enqueue_push(minife_ctx *c, int k, int mode, bool wait_now) {
    for (auto &p : c->parts) {
        const int64_t n = (int64_t)p.plan.send_idx.size();
        if (!n) continue;
        DevGuard g(p.dev);
        UpdArgs a = upd_args(c, p, 1);           // acc_in = rr_k (mode 1), p, r, rr, st
        LAUNCH(c, launch_push(a, k, mode, p.d_send_row, p.d_send_col, p.d_push_nbr, p.d_push_dst,
                              p.d_push_ptr, n, launch_stream(c, p)));
        if (c->mode == MINIFE_MODE_MULTI) CUDA_TRY(c, cudaEventRecord(p.ev_push, p.stream));
    }
    if (wait_now) return push_wait(c);
    return MINIFE_OK;
}

// Fill the halo (shell) columns of vec(part) from the owners' owned values.
// comm = true: on the transport streams (cstream) instead of the compute streams.
// prepacked = true: the send buffers already hold the values (k_pack_next_p); the wire
// protocol is used in every mode.
template <class VecOf>
static int enqueue_halo(minife_ctx *c, VecOf vec, bool comm = false, bool prepacked = false) {
    if (c->world == 1) return MINIFE_OK;
    // stream of part p's work: VIRTUAL ctxs use part 0's queue for every part
    auto sp = [&](Part &p) -> cudaStream_t {
        Part &q = c->mode == MINIFE_MODE_VIRTUAL ? c->parts[0] : p;
        return comm ? q.cstream : (c->mode == MINIFE_MODE_VIRTUAL ? q.stream : stream_of(c, q));
    };
    if (c->mode == MINIFE_MODE_VIRTUAL && c->transport == MINIFE_TRANSPORT_DIRECT && !prepacked) {
        // device-local transport: read the owner's columns through its send list, write the
        // receiver's halo columns
        cudaStream_t s = sp(c->parts[0]);
        for (auto &dst : c->parts) {
            for (size_t k = 0; k < dst.plan.nbr.size(); ++k) {
                Part &src = c->parts[dst.plan.nbr[k]];
                auto it = std::lower_bound(src.plan.nbr.begin(), src.plan.nbr.end(),
                                           dst.plan.rank);
                const size_t j = (size_t)(it - src.plan.nbr.begin());
                LAUNCH(c, launch_move(vec(src), src.d_send_col + src.plan.send_off[j], vec(dst),
                                        dst.d_recv_pos + dst.plan.recv_off[k],
                                        src.plan.send_cnt[j], s));
            }
        }
        return MINIFE_OK;
    }
    // wire protocol: pack each part's send lists, exchange per neighbor, unpack the slots
    for (auto &p : c->parts) {
        if (prepacked) break;
        DevGuard g(p.dev);
        LAUNCH(c, launch_move(vec(p), p.d_send_col, p.d_sendbuf, nullptr,
                                (int64_t)p.plan.send_idx.size(), sp(p)));
    }
    if (c->mode == MINIFE_MODE_VIRTUAL) {
        // loopback stand-in for ncclSend/ncclRecv: the bytes q sends to p land in p's receive
        // block for q, exactly where ncclRecv would put them
        cudaStream_t s = sp(c->parts[0]);
        for (auto &p : c->parts) {
            for (size_t k = 0; k < p.plan.nbr.size(); ++k) {
                Part &q = c->parts[p.plan.nbr[k]];
                auto it = std::lower_bound(q.plan.nbr.begin(), q.plan.nbr.end(), p.plan.rank);
                const size_t j = (size_t)(it - q.plan.nbr.begin());
                if (j >= q.plan.nbr.size() || q.plan.nbr[j] != p.plan.rank ||
                    q.plan.send_cnt[j] != p.plan.recv_cnt[k]) {
                    set_err(c, "halo plan mismatch between parts %d and %d", p.plan.rank,
                            q.plan.rank);
                    return MINIFE_ESTATE;
                }
                CUDA_TRY(c, cudaMemcpyAsync(p.d_recvbuf + p.plan.recv_off[k],
                                            q.d_sendbuf + q.plan.send_off[j],
                                            sizeof(double) * p.plan.recv_cnt[k],
                                            cudaMemcpyDeviceToDevice, s));
            }
        }
        for (auto &p : c->parts)
            LAUNCH(c, launch_move(p.d_recvbuf, nullptr, vec(p), p.d_recv_pos, p.plan.n_ext, s));
        return MINIFE_OK;
    }
    NCCL_TRY(c, nccl()->GroupStart());
    for (auto &p : c->parts) {
        cudaStream_t s = sp(p);
        for (size_t k = 0; k < p.plan.nbr.size(); ++k) {
            NCCL_TRY(c, nccl()->Send(p.d_sendbuf + p.plan.send_off[k],
                                     (size_t)p.plan.send_cnt[k], ncclFloat64, p.plan.nbr[k],
                                     p.comm, s));
            NCCL_TRY(c, nccl()->Recv(p.d_recvbuf + p.plan.recv_off[k],
                                     (size_t)p.plan.recv_cnt[k], ncclFloat64, p.plan.nbr[k],
                                     p.comm, s));
        }
    }
    NCCL_TRY(c, nccl()->GroupEnd());
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        LAUNCH(c, launch_move(p.d_recvbuf, nullptr, vec(p), p.d_recv_pos, p.plan.n_ext, sp(p)));
    }
    return MINIFE_OK;
}

// int64 SUM of the exact accumulators over all ranks (which = 0: pAp, 1: rr)
static int enqueue_allreduce(minife_ctx *c, int which, int k) {
    if (devcomm(c)) {           // every part stores its words into every rank's inbox
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            LAUNCH(c, launch_acc_push(upd_args(c, p, 0), k, which,
                                      which ? p.acc_rr() : p.acc_pAp(), launch_stream(c, p)));
        }
        return MINIFE_OK;
    }
    if (c->world == 1) return MINIFE_OK;
    if (c->mode == MINIFE_MODE_VIRTUAL) {
        std::vector<unsigned long long *> accs;
        for (auto &p : c->parts) accs.push_back(which ? p.acc_rr() : p.acc_pAp());
        LAUNCH(c, launch_vsum(accs.data(), (int)accs.size(), c->parts[0].stream));
        return MINIFE_OK;
    }
    NCCL_TRY(c, nccl()->GroupStart());
    for (auto &p : c->parts) {
        unsigned long long *a = which ? p.acc_rr() : p.acc_pAp();
        NCCL_TRY(c, nccl()->AllReduce(a, a, ACC_WORDS, ncclInt64, ncclSum, p.comm,
                                      stream_of(c, p)));
    }
    NCCL_TRY(c, nccl()->GroupEnd());
    return MINIFE_OK;
}

// ----------------------------------------------------------------------------------------
// CG driver (C6): init + max_iters x [halo, K1, reduce, K6, reduce, K7]
// ----------------------------------------------------------------------------------------

static UpdArgs upd_args(const minife_ctx *c, Part &p, int which_in) {
    UpdArgs a{};
    a.g = geom_of(c, p);
    a.x = p.d_x;
    a.r = p.d_r;
    a.p = p.d_p;
    a.Ap = p.d_Ap;
    a.b = p.d_b;
    a.hist = p.d_hist;
    a.rr = p.d_rr;
    a.st = p.d_st;
    a.x_late = c->opt.x_late;
    a.cl_dd = c->opt.cluster_dd;
    if (devcomm(c)) {
        a.rhalo = p.d_rhalo;
        a.halo_col = p.d_recv_pos;
        a.dc.region = p.d_comm_ptrs;
        a.dc.local = p.d_comm;
        a.dc.nbr_rank = p.d_nbr_rank;
        a.dc.n_nbr = (int)p.plan.nbr.size();
        a.dc.rank = p.plan.rank;
        a.dc.world = c->world;
        a.dc.timeout_ns = (long long)c->opt.comm_timeout_ms * 1000000ll;
        a.dc.mute = c->opt.comm_fault_part == p.plan.rank ? 1 : 0;
    }
    if (which_in == 0) {          // K6: in = pAp, out = rr
        a.acc_in = p.acc_pAp();
        a.acc_out = p.acc_rr();
        a.acc_zero = nullptr;
    } else {                      // K7: in = rr, zero pAp
        a.acc_in = p.acc_rr();
        a.acc_out = nullptr;
        a.acc_zero = p.acc_pAp();
    }
    return a;
}

// SYM storage per slice of 32 rows: 14 values, 9 run starts, 1 mask word per row
static constexpr int64_t SYM_SLICE_BYTES = 32 * (14 * 8 + 9 * 4 + 4);

// Snake order (odd iterations walk the SYM tiles backwards) where the matrix is within a few
// times the 126 MB L2: the tiles the previous SpMV read last are still resident when the next
// one starts there (B200, per solve: 80^3 (81 MB) -1 %, 100^3 (157 MB) -4 %, 120^3 (268 MB)
// -2 %, 150^3 none, 300^3 +2 %; profiles/r02/ab/snake_order.jsonl)
static bool snake_of(const minife_ctx *c, const Part &p) {
    if (c->opt.snake >= 0) return c->opt.snake > 0;
    const double bytes = (double)SYM_SLICE_BYTES * (double)p.nslices;
    return bytes > 48e6 && bytes < 400e6;
}

static SpmvArgs spmv_args(const minife_ctx *c, Part &p, const double *x, double *y, bool dot,
                          int k = 0) {
    SpmvArgs a{};
    a.m = matrix_of(c, p);
    a.g = geom_of(c, p);
    a.x = x;
    a.y = y;
    a.acc = dot ? p.acc_pAp() : nullptr;
    a.acc_zero = dot ? p.acc_rr() : nullptr;
    a.st = dot ? p.d_st : nullptr;
    a.s_begin = 0;
    a.s_end = a.m.nslices;
    // SYM value stream evict-first in L2 when the CG vectors (5 x 8 B per row) fit beside it
    // in the 126 MB L2 and so stay resident across the iteration's kernels (B200, 100^3:
    // 62.9 -> 60.9 us per iteration); at 300^3 the mirrored reads need the normal policy
    // (evict-first there: 1.207 -> 1.301 ms).  Option "val_evict_first" = 0/1 forces it.
    const int vef = c->opt.val_evict_first;
    a.val_evict_first = vef >= 0 ? vef : (40.0 * (double)p.ncols < 64e6 ? 1 : 0);
    // plane-ahead x prefetch into L2 when x itself does not stay L2-resident (B200, 300^3:
    // 1.0806 -> 1.0757 ms per iteration; 100^3: no gain).  Option "x_prefetch" = 0/1 forces it.
    const int xpf = c->opt.x_prefetch;
    a.x_prefetch = xpf >= 0 ? xpf : (8.0 * (double)p.ncols > 64e6 ? 1 : 0);
    a.sym_kernel = c->opt.sym_kernel;
    a.symm_nw = p.symm_nw;
    a.impl = c->opt.spmv_impl;
    a.tile_order = c->fmt == MINIFE_FMT_SYM ? p.d_tile_order : nullptr;
    // L2 reuse of the matrix across the solve's SpMVs (snake_of): the visiting order does not
    // change a bit of the result (every row's sum and the exact pAp are order-independent)
    a.reverse = c->fmt == MINIFE_FMT_SYM && dot && snake_of(c, p) && (k & 1);
    a.k = k;
    return a;
}

// Timing window: mark the start (end = false) or end of iteration k's SpMV on part 0's stream
static int tw_mark(minife_ctx *c, int k, bool end) {
    if (!c->tw_n || k < c->tw_k0 || k >= c->tw_k0 + c->tw_n) return MINIFE_OK;
    Part &p = c->parts[0];
    DevGuard g(p.dev);
    // External: a real event-record node when the stream is being captured into the graph
    // (a plain record when the solve is enqueued directly, MULTI ctxs or MINIFE_GRAPH=0)
    cudaStream_t s = launch_stream(c, p);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CUDA_TRY(c, cudaStreamIsCapturing(s, &cs));
    cudaEvent_t ev = c->tw_ev[2 * (k - c->tw_k0) + (end ? 1 : 0)];
    if (cs == cudaStreamCaptureStatusActive)
        CUDA_TRY(c, cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal));
    else
        CUDA_TRY(c, cudaEventRecord(ev, s));
    if (end && k == c->tw_k0 + c->tw_n - 1) c->tw_armed = true;
    return MINIFE_OK;
}

// The halo of p is moved on the parts' transport streams while the interior slices' SpMV
// runs (SEG, more than one part); the boundary slices follow once it has landed.
static bool overlap_mode(const minife_ctx *c) {
    return c->fmt == MINIFE_FMT_SEG && c->world > 1 && c->parts[0].cstream;
}

// SYM with a halo: the values p_(k+1) sends are computed ahead of K7 (k_pack_next_p); their
// exchange runs on the transport streams while K7 updates p, so the SpMV finds the halo in
// place.  (SYM stores rows by extended column, so the slices are not reordered.)
static bool overlap_sym(const minife_ctx *c) {
    return c->fmt == MINIFE_FMT_SYM && c->world > 1 && c->parts[0].cstream;
}

static int enqueue_k7_with_halo(minife_ctx *c, int k) {
    const bool virt = c->mode == MINIFE_MODE_VIRTUAL;
    if (push_mode(c)) {                  // device-initiated: p_(k+1) halo stored by the sender
        const bool last = k == c->cur_max_iters;     // no SpMV(k+1) reads it
        if (!last) TRY(enqueue_push(c, k, 1, false));
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            LAUNCH(c, launch_update_p(upd_args(c, p, 1), k, p.grid_upd, launch_stream(c, p)));
        }
        return last ? MINIFE_OK : push_wait(c);
    }
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        UpdArgs a = upd_args(c, p, 1);
        LAUNCH(c, launch_pack_next_p(a, k, p.d_send_row, p.d_send_col, p.d_sendbuf,
                                       (int64_t)p.plan.send_idx.size(), launch_stream(c, p)));
    }
    for (auto &p : c->parts) {
        if (virt && &p != &c->parts[0]) break;
        DevGuard g(p.dev);
        CUDA_TRY(c, cudaEventRecord(p.ev_fork, launch_stream(c, p)));
        CUDA_TRY(c, cudaStreamWaitEvent(p.cstream, p.ev_fork, 0));
    }
    TRY(enqueue_halo(c, [](Part &p) { return p.d_p; }, true, true));
    for (auto &p : c->parts) {
        if (virt && &p != &c->parts[0]) break;
        DevGuard g(p.dev);
        CUDA_TRY(c, cudaEventRecord(p.ev_join, p.cstream));
    }
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        LAUNCH(c, launch_update_p(upd_args(c, p, 1), k, p.grid_upd, launch_stream(c, p)));
    }
    for (auto &p : c->parts) {
        if (virt && &p != &c->parts[0]) break;
        DevGuard g(p.dev);
        CUDA_TRY(c, cudaStreamWaitEvent(launch_stream(c, p), p.ev_join, 0));
    }
    return MINIFE_OK;
}

struct PhaseTimer {
    std::vector<cudaEvent_t> ev;
    std::vector<int> phase;     // phase of the interval ending at ev[i]
    cudaStream_t s = nullptr;
    void mark(int ph) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.push_back(e);
        phase.push_back(ph);
    }
};

// Halo by r (device comm): r_(kp) at every part's send slots into the receivers' r-halo
// buffers, flags raised by the last CTA (kp = k + 1 after K6(k); kp = 1 at init: r_0 = b)
static int enqueue_push_r(minife_ctx *c, int kp) {
    for (auto &p : c->parts) {
        const int64_t n = (int64_t)p.plan.send_idx.size();
        if (!n) continue;
        DevGuard g(p.dev);
        LAUNCH(c, launch_push_r(upd_args(c, p, 1), kp, p.d_send_row, p.d_push_nbr, p.d_rdst,
                                p.d_rhalo_ptr, n, launch_stream(c, p)));
    }
    return MINIFE_OK;
}

static int enqueue_init(minife_ctx *c, double tol) {
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        cudaStream_t s = launch_stream(c, p);
        CUDA_TRY(c, cudaMemsetAsync(p.d_acc, 0, 4 * ACC_WORDS * sizeof(unsigned long long), s));
        UpdArgs a = upd_args(c, p, 0);
        a.acc_out = p.acc_rr();
        a.fold_push = fold_comm(c) ? 1 : 0;          // the last CTA pushes rr_0
        LAUNCH(c, launch_init_vectors(a, p.grid_upd, s));
    }
    if (!fold_comm(c)) TRY(enqueue_allreduce(c, 1, 0));
    if (devcomm(c)) TRY(enqueue_push_r(c, 1));      // r_0 = b at the send slots (p_1's halo)
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        UpdArgs a = upd_args(c, p, 0);
        a.acc_out = p.acc_rr();
        a.acc_zero = p.acc_pAp();
        LAUNCH(c, launch_init_finalize(a, tol, launch_stream(c, p)));
    }
    if (devcomm(c))
        for (auto &p : c->parts) {                   // p_1's halo columns = r_0's halo
            if (!p.plan.n_ext) continue;
            DevGuard g(p.dev);
            UpdArgs a = upd_args(c, p, 0);
            a.halo_n = p.plan.n_ext;
            LAUNCH(c, launch_halo_init(a, launch_stream(c, p)));
        }
    return MINIFE_OK;
}

// a1 + a2 with the halo in flight during the interior SpMV: fork the transport streams off
// the compute streams (p is final after K7), interior slices, join, boundary slices.  The
// pAp accumulator is order-independent (C5), so the split changes no bit of the result.
static int enqueue_halo_spmv_overlapped(minife_ctx *c, int k) {
    const bool virt = c->mode == MINIFE_MODE_VIRTUAL;
    for (auto &p : c->parts) {
        if (virt && &p != &c->parts[0]) break;
        DevGuard g(p.dev);
        CUDA_TRY(c, cudaEventRecord(p.ev_fork, launch_stream(c, p)));
        CUDA_TRY(c, cudaStreamWaitEvent(p.cstream, p.ev_fork, 0));
    }
    TRY(enqueue_halo(c, [](Part &p) { return p.d_p; }, true));
    for (auto &p : c->parts) {
        if (virt && &p != &c->parts[0]) break;
        DevGuard g(p.dev);
        CUDA_TRY(c, cudaEventRecord(p.ev_join, p.cstream));
    }
    TRY(tw_mark(c, k, false));
    for (auto &p : c->parts) {                     // interior slices: no halo column read
        DevGuard g(p.dev);
        SpmvArgs a = spmv_args(c, p, p.d_p, p.d_Ap, true);
        a.s_end = p.n_int;
        if (a.s_end > a.s_begin) LAUNCH(c, launch_spmv(a, true, p.grid_spmv, launch_stream(c, p)));
    }
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        Part &q = virt ? c->parts[0] : p;
        if (!virt || &p == &c->parts[0])
            CUDA_TRY(c, cudaStreamWaitEvent(launch_stream(c, p), q.ev_join, 0));
        SpmvArgs a = spmv_args(c, p, p.d_p, p.d_Ap, true);
        a.s_begin = p.n_int;
        if (a.s_end > a.s_begin) LAUNCH(c, launch_spmv(a, true, p.grid_spmv, launch_stream(c, p)));
    }
    TRY(tw_mark(c, k, true));
    return MINIFE_OK;
}

static int enqueue_iteration(minife_ctx *c, int k, PhaseTimer *t) {
    const bool osym = overlap_sym(c) && !t;
    if (overlap_mode(c) && !t && !push_mode(c)) {
        TRY(enqueue_halo_spmv_overlapped(c, k));
    } else if (osym) {                               // halo already in place (previous K7)
        TRY(tw_mark(c, k, false));
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            SpmvArgs sa = spmv_args(c, p, p.d_p, p.d_Ap, true, k);
            if (fold_comm(c)) {                      // the SpMV's last CTA pushes pAp_k
                sa.dc = upd_args(c, p, 0).dc;
                sa.fold_push = 1;
                sa.k = k;
            }
            LAUNCH(c, launch_spmv(sa, true, p.grid_spmv, launch_stream(c, p)));
        }
        TRY(tw_mark(c, k, true));
    } else {
        if (push_mode(c)) TRY(enqueue_push(c, k, 0, true));
        else TRY(enqueue_halo(c, [](Part &p) { return p.d_p; }));
        if (t) t->mark(3);
        if (!t) TRY(tw_mark(c, k, false));
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            LAUNCH(c, launch_spmv(spmv_args(c, p, p.d_p, p.d_Ap, true, k), true, p.grid_spmv,
                                    launch_stream(c, p)));
        }
        if (!t) TRY(tw_mark(c, k, true));
    }
    if (t) t->mark(0);
    if (!(osym && fold_comm(c))) TRY(enqueue_allreduce(c, 0, k));
    if (t) t->mark(3);
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        UpdArgs u6 = upd_args(c, p, 0);
        u6.fold_push = fold_comm(c) ? 1 : 0;          // K6's last CTA pushes rr_k
        LAUNCH(c, launch_update_xr(u6, k, p.grid_upd, launch_stream(c, p)));
    }
    if (t) t->mark(1);
    if (!fold_comm(c)) TRY(enqueue_allreduce(c, 1, k));
    if (t) t->mark(3);
    if (osym) {
        TRY(enqueue_k7_with_halo(c, k));
    } else {
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            LAUNCH(c, launch_update_p(upd_args(c, p, 1), k, p.grid_upd, launch_stream(c, p)));
        }
    }
    if (t) t->mark(2);
    return MINIFE_OK;
}

static int ensure_hist(minife_ctx *c, int max_iters) {
    if (c->parts[0].hist_cap >= max_iters + 1) return MINIFE_OK;
    for (auto &p : c->parts) TRY(alloc_hist(c, p, max_iters + 1));
    drop_graph(c);
    return MINIFE_OK;
}

// Fused two-kernel iteration: one part, SEG format,
// selected with minife_set_scheme (default: the three-kernel sequence, faster on B200 today,
// profiles/r01).  Both schemes give the same results, bit for bit.
static bool fused_mode(const minife_ctx *c) {
    return c->scheme == MINIFE_SCHEME_FUSED && c->parts.size() == 1 &&
           c->fmt == MINIFE_FMT_SEG && c->parts[0].ncols == c->parts[0].rows;
}

static int enqueue_iteration_fused(minife_ctx *c, int k, PhaseTimer *t) {
    Part &p = c->parts[0];
    DevGuard g(p.dev);
    cudaStream_t s = launch_stream(c, p);
    // F1(k): p_k = r + beta_{k-1} p_{k-1} at gather time, Ap_k, exact pAp_k, deferred x
    SpmvArgs a = spmv_args(c, p, p.p_buf(k - 1), p.d_Ap, true);
    a.acc = p.acc_pAp(k);
    a.acc_zero = p.acc_rr(k);            // read by F1(k-1): free for K6'(k)
    a.fused_k = k;
    a.r = p.d_r;
    a.p_old = p.p_buf(k - 1);
    a.p_new = p.p_buf(k);
    a.xsol = p.d_x;
    a.acc_rr_in = p.acc_rr(k - 1);
    a.hist = p.d_hist;
    a.rr = p.d_rr;
    a.stw = p.d_st;
    if (!t) TRY(tw_mark(c, k, false));
    LAUNCH(c, launch_spmv(a, true, p.grid_spmv, s));
    if (!t) TRY(tw_mark(c, k, true));
    if (t) t->mark(0);
    // K6'(k): alpha_k, r -= alpha_k Ap_k, exact rr_k
    UpdArgs u = upd_args(c, p, 0);
    u.acc_in = p.acc_pAp(k);
    u.acc_out = p.acc_rr(k);
    LAUNCH(c, launch_update_r(u, k, p.acc_pAp(k + 1), p.grid_upd, s));
    if (t) t->mark(1);
    return MINIFE_OK;
}

// init + max_iters iterations (+ the fused scheme's finish kernel), enqueued on the streams
// x every second iteration (one part, three-kernel scheme): K7 of an odd iteration leaves x
// alone and writes p_(k+1) into the other p buffer; the next (even) K7 applies
// alpha_(k-1) p_(k-1) and alpha_k p_k in one pass over x.  x then costs 16 B per row every
// second iteration (36 instead of 40 B/row per K7 on average); same operations, same order:
// bit-identical.
// Deferred x: x += alpha_k p_k is applied X iterations at a time, p_k living
// in a ring of X buffers.  Returns X, or 0 when off.  Option "x_defer" = 0 disables it, n
// (2..8) forces X = n at any size (tests); -1 (default): X = XDEF_DEFAULT where the vectors stream
// from HBM anyway (B200, 300^3 per iteration: X = 2 -1.0 % against no deferral, X = 4 a
// further -0.5 %, X = 8 -1.1 %; K7 moves 24 B/row plus (16 + 8 (X-1)) / X for x; at 100^3,
// whose vectors sit in L2, a second p buffer costs +0.7 %).
constexpr int XDEF_DEFAULT = 8;
static int xdef_of(const minife_ctx *c) {
    const int env = c->opt.x_defer;
    // partitioned (SYM with a halo, halo overlapped with K7 over the wire or device copies):
    // the exchange fills the halo of the buffer p_(k+1) goes to
    const bool single = c->parts.size() == 1 && c->world == 1;
    // (device comm: each part completes the halo columns of p_(k+1) in the ring buffer itself)
    const bool parts_ok = overlap_sym(c) && !push_mode(c);
    if (!env || env == 1 || !(single || parts_ok) || fused_mode(c)) return 0;
    if (env >= 2) return std::min(env, XDEF_MAX);
    // automatic: single parts only -- on partitioned parts (x-line walks, halo exchange each
    // iteration) the deferral is slower: B200, 2 virtual parts of 600x300x300 2.133 vs 2.079
    // ms per iteration, 8 parts of 400^3 2.640 vs 2.595 (profiles/r02/ab)
    return single && 40.0 * (double)c->parts[0].ncols >= 64e6 ? XDEF_DEFAULT : 0;
}
static bool x2_mode(const minife_ctx *c) { return xdef_of(c) > 0; }

static int ensure_fused_buffers(minife_ctx *c) {   // never called while a stream captures
    if (!(fused_mode(c) || x2_mode(c))) return MINIFE_OK;
    const int X = std::max(2, xdef_of(c));
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        if (!p.d_p2) TRY(alloc_colvec(c, p, &p.d_p2));
        for (int i = 2; i < X; ++i)
            if (!p.d_pr[i]) TRY(alloc_colvec(c, p, &p.d_pr[i]));
    }
    return MINIFE_OK;
}

// Single-launch solvers for small single-part problems (SEG/SYM): 0 = none, 1 = one CTA
// (k_cg_small, <= SMALL_MAX_ROWS rows), 2 = one thread-block cluster (k_cg_cluster, <=
// CL_MAX_ROWS rows).  Option "small_solver" = 0/1/2 forces a choice (where it fits).  Profile
// mode always times the multi-kernel sequence.
static bool cluster_available(const Part &p) {
    DevGuard g(p.dev);
    return cluster_solver_available();
}
static int small_mode(const minife_ctx *c) {
    const int env = c->opt.small_solver;
    const Part &p = c->parts[0];
    if (env == 0 || c->parts.size() != 1 || c->world != 1 || p.ncols != p.rows ||
        (c->fmt != MINIFE_FMT_SEG && c->fmt != MINIFE_FMT_SYM))
        return 0;
    const bool fits1 = p.rows <= SMALL_MAX_ROWS;
    const bool fits2 = p.rows <= CL_MAX_ROWS &&
                       (p.nslices + CL_CTAS - 1) / CL_CTAS <= CL_MAX_SL && cluster_available(p);
    if (env == 1) return fits1 ? 1 : 0;
    if (env == 2) return fits2 ? 2 : 0;
    return fits2 ? 2 : (fits1 ? 1 : 0);
}

// p_k of the x-every-2 scheme: p_1 (written by the init kernels) in d_p, then alternating
static double *x2_pbuf(const minife_ctx *c, const Part &p, int k) {
    return p.ring((k - 1) % xdef_of(c));
}
static void set_ring(const minife_ctx *c, const Part &p, UpdArgs &u) {
    const int X = xdef_of(c);
    for (int i = 0; i < XDEF_MAX; ++i) u.ring[i] = i < X ? p.ring(i) : nullptr;
    u.xdef = X;
}

static int enqueue_iteration_x2(minife_ctx *c, int k) {
    const bool virt = c->mode == MINIFE_MODE_VIRTUAL;
    const bool halo = c->parts.size() > 1 || c->world > 1;
    const bool fold = fold_comm(c);
    TRY(tw_mark(c, k, false));
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        SpmvArgs sa = spmv_args(c, p, x2_pbuf(c, p, k), p.d_Ap, true, k);
        if (fold) {                                  // the SpMV's last CTA pushes pAp_k
            sa.dc = upd_args(c, p, 0).dc;
            sa.fold_push = 1;
            sa.k = k;
        }
        LAUNCH(c, launch_spmv(sa, true, p.grid_spmv, launch_stream(c, p)));
    }
    TRY(tw_mark(c, k, true));
    if (!fold) TRY(enqueue_allreduce(c, 0, k));
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        UpdArgs u6 = upd_args(c, p, 0);
        u6.alpha_hist = p.d_alpha;
        u6.fold_push = fold ? 1 : 0;
        LAUNCH(c, launch_update_xr(u6, k, p.grid_upd, launch_stream(c, p)));
    }
    if (!fold) TRY(enqueue_allreduce(c, 1, k));
    if (halo) {
        // as enqueue_k7_with_halo: the send slots' p_(k+1) ahead of K7, exchanged on the
        // transport stream into the halo of the buffer p_(k+1) goes to, while K7 runs
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            UpdArgs a = upd_args(c, p, 1);
            a.p = x2_pbuf(c, p, k);
            LAUNCH(c, launch_pack_next_p(a, k, p.d_send_row, p.d_send_col, p.d_sendbuf,
                                           (int64_t)p.plan.send_idx.size(), launch_stream(c, p)));
        }
        for (auto &p : c->parts) {
            if (virt && &p != &c->parts[0]) break;
            DevGuard g(p.dev);
            CUDA_TRY(c, cudaEventRecord(p.ev_fork, launch_stream(c, p)));
            CUDA_TRY(c, cudaStreamWaitEvent(p.cstream, p.ev_fork, 0));
        }
        TRY(enqueue_halo(c, [c, k](Part &p) { return x2_pbuf(c, p, k + 1); }, true, true));
        for (auto &p : c->parts) {
            if (virt && &p != &c->parts[0]) break;
            DevGuard g(p.dev);
            CUDA_TRY(c, cudaEventRecord(p.ev_join, p.cstream));
        }
    }
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        UpdArgs u7 = upd_args(c, p, 1);
        u7.alpha_hist = p.d_alpha;
        set_ring(c, p, u7);
        LAUNCH(c, launch_update_p2(u7, k, x2_pbuf(c, p, k), x2_pbuf(c, p, k + 1), p.grid_upd,
                                     launch_stream(c, p)));
    }
    if (halo) {
        for (auto &p : c->parts) {
            if (virt && &p != &c->parts[0]) break;
            DevGuard g(p.dev);
            CUDA_TRY(c, cudaStreamWaitEvent(launch_stream(c, p), p.ev_join, 0));
        }
    }
    return MINIFE_OK;
}

// Device-initiated comm: per iteration SpMV (its last CTA pushes pAp_k) |
// K6 (its last CTA pushes rr_k) | the halo push of r_(k+1) (needs no reduction result, so it
// overlaps the rr reduction) | K7, which also completes p_(k+1)'s halo columns from the
// neighbours' r_(k+1).  With or without the deferred-x ring; profile mode marks the phases.
static int enqueue_solve_dev(minife_ctx *c, int max_iters, double tol, PhaseTimer *t) {
    const int X = t ? 0 : xdef_of(c);
    const bool fold = fold_comm(c);
    TRY(enqueue_init(c, tol));
    if (t) t->mark(-1);
    for (int k = 1; k <= max_iters; ++k) {
        const bool last = k == max_iters;
        if (!t) TRY(tw_mark(c, k, false));
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            SpmvArgs sa = spmv_args(c, p, X ? x2_pbuf(c, p, k) : p.d_p, p.d_Ap, true, k);
            if (fold) {                              // the SpMV's last CTA pushes pAp_k
                sa.dc = upd_args(c, p, 0).dc;
                sa.fold_push = 1;
                sa.k = k;
            }
            LAUNCH(c, launch_spmv(sa, true, p.grid_spmv, launch_stream(c, p)));
        }
        if (!t) TRY(tw_mark(c, k, true));
        if (t) t->mark(0);
        if (!fold) TRY(enqueue_allreduce(c, 0, k));
        if (t) t->mark(3);
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            UpdArgs u6 = upd_args(c, p, 0);
            if (X) u6.alpha_hist = p.d_alpha;
            u6.fold_push = fold ? 1 : 0;             // K6's last CTA pushes rr_k
            LAUNCH(c, launch_update_xr(u6, k, p.grid_upd, launch_stream(c, p)));
        }
        if (t) t->mark(1);
        if (!fold) TRY(enqueue_allreduce(c, 1, k));
        if (!last) TRY(enqueue_push_r(c, k + 1));
        if (t) t->mark(3);
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            UpdArgs u7 = upd_args(c, p, 1);
            if (!last && p.plan.n_ext) {             // p_(k+1)'s halo columns, from r_(k+1)
                u7.halo_n = p.plan.n_ext;
                u7.halo_kp = k + 1;
            }
            if (X) {
                u7.alpha_hist = p.d_alpha;
                set_ring(c, p, u7);
                LAUNCH(c, launch_update_p2(u7, k, x2_pbuf(c, p, k), x2_pbuf(c, p, k + 1),
                                           p.grid_upd, launch_stream(c, p)));
            } else {
                LAUNCH(c, launch_update_p(u7, k, p.grid_upd, launch_stream(c, p)));
            }
        }
        if (t) t->mark(2);
    }
    if (X)
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            UpdArgs u = upd_args(c, p, 0);
            u.alpha_hist = p.d_alpha;
            set_ring(c, p, u);
            LAUNCH(c, launch_x2_finish(u, launch_stream(c, p)));
        }
    return MINIFE_OK;
}

static int enqueue_solve(minife_ctx *c, int max_iters, double tol, PhaseTimer *t) {
    if (!t) c->tw_armed = false;
    c->cur_max_iters = max_iters;
    if (devcomm(c) && !small_mode(c) && !fused_mode(c)) return enqueue_solve_dev(c, max_iters, tol, t);
    if (!t && x2_mode(c) && !small_mode(c)) {
        TRY(enqueue_init(c, tol));
        if (c->parts.size() > 1 || c->world > 1) {    // halo of p_1 = b (buffer of odd k)
            TRY(enqueue_halo(c, [](Part &p) { return p.d_p; }));
        }
        for (int k = 1; k <= max_iters; ++k) TRY(enqueue_iteration_x2(c, k));
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            UpdArgs u = upd_args(c, p, 0);
            u.alpha_hist = p.d_alpha;
            set_ring(c, p, u);
            LAUNCH(c, launch_x2_finish(u, launch_stream(c, p)));
        }
        return MINIFE_OK;
    }
    const int sm = t ? 0 : small_mode(c);
    if (sm) {
        Part &p = c->parts[0];
        DevGuard g(p.dev);
        if (sm == 1)
            LAUNCH(c, launch_cg_small(matrix_of(c, p), upd_args(c, p, 0), max_iters, tol,
                                        launch_stream(c, p)));
        else
            LAUNCH(c, launch_cg_cluster(matrix_of(c, p), upd_args(c, p, 0), max_iters, tol,
                                          launch_stream(c, p)));
        return MINIFE_OK;
    }
    const bool fused = fused_mode(c);
    TRY(enqueue_init(c, tol));
    if (!t && overlap_sym(c)) {                      // halo of p_1 = b
        if (push_mode(c)) TRY(enqueue_push(c, 0, 0, true));
        else TRY(enqueue_halo(c, [](Part &p) { return p.d_p; }));
    }
    if (t) t->mark(-1);
    for (int k = 1; k <= max_iters; ++k)
        TRY(fused ? enqueue_iteration_fused(c, k, t) : enqueue_iteration(c, k, t));
    if (fused) {
        Part &p = c->parts[0];
        DevGuard g(p.dev);
        UpdArgs u = upd_args(c, p, 0);
        u.acc_in = p.acc_rr(max_iters);
        LAUNCH(c, launch_cg_finish(u, max_iters, p.p_buf(0), p.p_buf(1), p.grid_upd,
                                     launch_stream(c, p)));
        if (t) t->mark(2);
    }
    return MINIFE_OK;
}

static double spmv_alg_bytes(const minife_ctx *c, const Part &q) {
    // CRS 12 nnz (+16 rows of x/y); segment format 8 nnz + 4 nns (+16 rows)
    // SYM: values of the upper triangle incl. the diagonal, (nnz + rows) / 2
    if (c->fmt == MINIFE_FMT_SYM)
        return 8.0 * 0.5 * (double)(q.nnz + q.rows) + 4.0 * (double)q.nns;
    return c->fmt == MINIFE_FMT_CRS ? 12.0 * (double)q.nnz
                                    : 8.0 * (double)q.nnz + 4.0 * (double)q.nns;
}

static int read_result(minife_ctx *c, int max_iters, minife_cg_result *res, double seconds) {
    Part &p = c->parts[0];
    DevGuard g(p.dev);
    CgState st;
    double h0 = 0.0;
    CUDA_TRY(c, cudaMemcpy(&st, p.d_st, sizeof st, cudaMemcpyDeviceToHost));
    CUDA_TRY(c, cudaMemcpy(&h0, p.d_hist, sizeof h0, cudaMemcpyDeviceToHost));
    double hk = h0;
    if (st.iters > 0)
        CUDA_TRY(c, cudaMemcpy(&hk, p.d_hist + st.iters, sizeof hk, cudaMemcpyDeviceToHost));
    c->last_iters = st.iters;
    c->solved = true;
    const int status = st.status == 6 ? MINIFE_ENOTSPD
                       : st.status == 7 ? MINIFE_EDIVERGED
                       : st.status == 9 ? MINIFE_ECOMM
                                        : MINIFE_OK;
    if (status == MINIFE_ECOMM)
        set_err(c, "device comm: a peer did not signal within %d ms", c->opt.comm_timeout_ms);
    if (res) {
        res->status = status;
        res->iterations = st.iters;
        res->converged = st.converged;
        res->max_iters = max_iters;
        res->norm_b = h0;
        res->final_rel_residual = h0 > 0.0 ? hk / h0 : 0.0;
        res->seconds = seconds;
        const double rows = (double)c->mesh.rows(), nnz = (double)c->mesh.nnz();
        res->flops = (double)st.iters * (2.0 * nnz + 10.0 * rows);
        // vector bytes per row: 80 (three-kernel scheme, x updated with p), 76 (x every
        // second iteration: K7 moves 24 and 48 B/row alternately) or 72 (fused)
        const int X = xdef_of(c);
        const double vec = fused_mode(c) ? 72.0 : (X && !small_mode(c) ? 72.0 + 8.0 / X : 80.0);
        double bytes = 0.0;
        for (auto &q : c->parts) bytes += spmv_alg_bytes(c, q) + vec * (double)q.rows;
        res->bytes = (double)st.iters * bytes;
    }
    return status;
}

static int check_solve_args(minife_ctx *c, int max_iters, double tol) {
    if (!c) return MINIFE_EINVAL;
    if (!c->assembled) {
        set_err(c, "minife_cg_solve before minife_assemble");
        return MINIFE_ESTATE;
    }
    if (max_iters < 1 || !(tol >= 0.0)) return MINIFE_EINVAL;
    return ensure_fused_buffers(c);
}

// Wait for the end of an enqueued solve.  With NCCL comms, poll ncclCommGetAsyncError while
// waiting: a failed or dead peer surfaces as MINIFE_ENCCL (communicators aborted) instead of a
// hang.
static int wait_solve(minife_ctx *c, cudaEvent_t done) {
    bool any_comm = false;
    for (auto &p : c->parts) any_comm |= p.comm != nullptr;
    if (!any_comm || !nccl()->CommGetAsyncError) {
        CUDA_TRY(c, cudaEventSynchronize(done));
        return MINIFE_OK;
    }
    for (;;) {
        const cudaError_t q = cudaEventQuery(done);
        if (q == cudaSuccess) return MINIFE_OK;
        if (q != cudaErrorNotReady) CUDA_TRY(c, q);
        for (auto &p : c->parts) {
            if (!p.comm) continue;
            ncclResult_t ae = ncclSuccess;
            if (nccl()->CommGetAsyncError(p.comm, &ae) != ncclSuccess || ae != ncclSuccess) {
                set_err(c, "NCCL asynchronous error: %s", nccl()->GetErrorString(ae));
                for (auto &q2 : c->parts)
                    if (q2.comm) {
                        nccl()->CommAbort(q2.comm);
                        q2.comm = nullptr;
                    }
                return MINIFE_ENCCL;
            }
        }
        struct timespec ts = {0, 50000};
        nanosleep(&ts, nullptr);
    }
}

extern "C" int minife_cg_solve(minife_ctx *c, int max_iters, double tol, minife_cg_result *res) {
    NvtxRange nvtx_("minife_cg_solve");
    TRY(check_solve_args(c, max_iters, tol));
    TRY(ensure_hist(c, max_iters));
    Part &p0 = c->parts[0];
    DevGuard g(p0.dev);
    // MULTI with device comm: one graph per device (no cross-device dependency other than the
    // in-kernel flags); MULTI with NCCL reductions: enqueued directly.  Option "graph" = 0:
    // enqueue every solve directly (an escape hatch should capturing NCCL calls fail).
    const bool per_part = c->mode == MINIFE_MODE_MULTI && devcomm(c);
    bool eager = (c->mode == MINIFE_MODE_MULTI && !per_part) || !c->opt.graph || c->eager;
    const bool have = per_part ? !c->gexec_parts.empty() : c->gexec != nullptr;
    if (!eager && (!have || c->g_iters != max_iters || c->g_tol != tol)) {
        drop_graph(c);
        // capture on the ctx's own streams (a torch stream may be the legacy default one)
        cudaStream_t saved = c->user_stream;
        c->user_stream = nullptr;
        std::vector<cudaStream_t> caps;
        if (per_part)
            for (auto &p : c->parts) caps.push_back(p.stream);
        else
            caps.push_back(p0.stream);
        cudaError_t e = cudaSuccess;
        size_t begun = 0;
        for (size_t i = 0; i < caps.size() && e == cudaSuccess; ++i) {
            DevGuard gg(per_part ? c->parts[i].dev : p0.dev);
            e = cudaStreamBeginCapture(caps[i], cudaStreamCaptureModeThreadLocal);
            if (e == cudaSuccess) ++begun;
        }
        const int64_t k0 = c->enq_kernels;
        int st = e == cudaSuccess ? enqueue_solve(c, max_iters, tol, nullptr) : MINIFE_OK;
        const int64_t captured = c->enq_kernels - k0;
        c->enq_kernels = k0;
        std::vector<cudaGraphExec_t> execs;
        for (size_t i = 0; i < begun; ++i) {
            DevGuard gg(per_part ? c->parts[i].dev : p0.dev);
            cudaGraph_t graph = nullptr;
            cudaError_t e2 = cudaStreamEndCapture(caps[i], &graph);
            if (e == cudaSuccess) e = e2;
            cudaGraphExec_t ex = nullptr;
            if (st == MINIFE_OK && e == cudaSuccess) {
                e = cudaGraphInstantiate(&ex, graph, 0);
                if (e == cudaSuccess) execs.push_back(ex);
            }
            if (graph) cudaGraphDestroy(graph);
        }
        c->user_stream = saved;
        if (st != MINIFE_OK || e != cudaSuccess || execs.size() != caps.size()) {
            for (auto ex : execs) cudaGraphExecDestroy(ex);
            // a multi-rank job whose capture failed (every rank takes the same path) runs
            // this and later solves directly; anything else is an error
            if (c->world > 1 && (c->mode == MINIFE_MODE_RANK || per_part)) {
                cudaGetLastError();
                c->eager = eager = true;
            } else {
                if (st != MINIFE_OK) return st;
                CUDA_TRY(c, e != cudaSuccess ? e : cudaErrorUnknown);
            }
        } else {
            if (per_part) c->gexec_parts = execs;
            else c->gexec = execs[0];
            c->g_iters = max_iters;
            c->g_tol = tol;
            c->g_kernels = captured;
        }
    }
    TRY(mark_parts(c, false));
    if (eager) {
        // one host thread drives every device: launch the sequence directly
        TRY(enqueue_solve(c, max_iters, tol, nullptr));
    } else if (per_part) {
        for (size_t i = 0; i < c->parts.size(); ++i) {
            DevGuard gg(c->parts[i].dev);
            CUDA_TRY(c, cudaGraphLaunch(c->gexec_parts[i], c->parts[i].stream));
        }
        c->kernel_launches += c->g_kernels;
    } else {
        CUDA_TRY(c, cudaGraphLaunch(c->gexec, launch_stream(c, p0)));
        c->kernel_launches += c->g_kernels;
    }
    TRY(mark_parts(c, true));
    for (auto &p : c->parts) {
        DevGuard gg(p.dev);
        TRY(wait_solve(c, p.ev_t1));
    }
    TRY(elapsed_parts(c, &c->last_solve_ms, &Part::t_solve_ms));
    return read_result(c, max_iters, res, c->last_solve_ms * 1e-3);
}

extern "C" int minife_set_timing_window(minife_ctx *c, int first_iter, int n_iters) {
    if (!c || first_iter < 1 || n_iters < 0) return MINIFE_EINVAL;
    DevGuard g(c->parts[0].dev);
    for (cudaEvent_t e : c->tw_ev) cudaEventDestroy(e);
    c->tw_ev.assign(2 * (size_t)n_iters, nullptr);
    for (auto &e : c->tw_ev) CUDA_TRY(c, cudaEventCreate(&e));
    c->tw_k0 = first_iter;
    c->tw_n = n_iters;
    drop_graph(c);
    return MINIFE_OK;
}

extern "C" int minife_get_timing_window(minife_ctx *c, double *spmv_ms, double *iter_ms) {
    if (!c || !spmv_ms || !iter_ms) return MINIFE_EINVAL;
    if (!c->tw_n || !c->tw_armed || !c->solved || c->last_iters < c->tw_k0 + c->tw_n - 1) {
        set_err(c, "no solve has run through the whole timing window (single-launch solvers "
                   "have none)");
        return MINIFE_ESTATE;
    }
    DevGuard g(c->parts[0].dev);
    double sum = 0.0;
    for (int j = 0; j < c->tw_n; ++j) {
        float ms = 0.f;
        const cudaError_t e = cudaEventElapsedTime(&ms, c->tw_ev[2 * j], c->tw_ev[2 * j + 1]);
        if (e != cudaSuccess) {
            cudaGetLastError();                  // not sticky: do not poison later launches
            set_err(c, "cudaEventElapsedTime on the timing window: %s", cudaGetErrorString(e));
            return MINIFE_ECUDA;
        }
        sum += ms;
    }
    *spmv_ms = sum / c->tw_n;
    *iter_ms = 0.0;
    if (c->tw_n >= 2) {
        float ms = 0.f;
        const cudaError_t e = cudaEventElapsedTime(&ms, c->tw_ev[0], c->tw_ev[2 * (c->tw_n - 1)]);
        if (e != cudaSuccess) {
            cudaGetLastError();
            set_err(c, "cudaEventElapsedTime on the timing window: %s", cudaGetErrorString(e));
            return MINIFE_ECUDA;
        }
        *iter_ms = ms / (c->tw_n - 1);
    }
    return MINIFE_OK;
}

extern "C" int minife_cg_profile(minife_ctx *c, int max_iters, minife_kernel_times *out) {
    NvtxRange nvtx_("minife_cg_profile");
    TRY(check_solve_args(c, max_iters, 0.0));
    TRY(ensure_hist(c, max_iters));
    Part &p0 = c->parts[0];
    DevGuard g(p0.dev);
    PhaseTimer t;
    t.s = launch_stream(c, p0);
    TRY(enqueue_solve(c, max_iters, 0.0, &t));
    for (auto &p : c->parts) {
        DevGuard gg(p.dev);
        CUDA_TRY(c, cudaStreamSynchronize(launch_stream(c, p)));
    }
    double ms[4] = {0, 0, 0, 0};
    for (size_t i = 1; i < t.ev.size(); ++i) {
        float m = 0.f;
        cudaEventElapsedTime(&m, t.ev[i - 1], t.ev[i]);
        if (t.phase[i] >= 0) ms[t.phase[i]] += m;
    }
    for (auto e : t.ev) cudaEventDestroy(e);
    if (out) {
        out->spmv_ms = ms[0];
        out->update_xr_ms = ms[1];
        out->update_p_ms = ms[2];
        out->comm_ms = ms[3];
        out->spmv_launches = out->update_xr_launches = max_iters;
        out->update_p_launches = fused_mode(c) ? 1 : max_iters;   // fused: the finish kernel
        out->iterations = max_iters;
    }
    return read_result(c, max_iters, nullptr, 0.0);
}

// ----------------------------------------------------------------------------------------
// host <-> part index helpers
// ----------------------------------------------------------------------------------------

static int64_t gid_of_row(const Plan &pl, int64_t l) {
    const int64_t lx = l % pl.own_n[0], ly = (l / pl.own_n[0]) % pl.own_n[1],
                  lz = l / (pl.own_n[0] * pl.own_n[1]);
    return (pl.own_lo[0] + lx) +
           pl.mesh.NX() * ((pl.own_lo[1] + ly) + pl.mesh.NY() * (pl.own_lo[2] + lz));
}

// global <-> owned-local scatter/gather on the host (box enumeration, x-lines contiguous)
static void gather_owned(const Plan &pl, const double *global, double *local) {
    const int64_t NX = pl.mesh.NX(), NY = pl.mesh.NY();
    int64_t l = 0;
    for (int64_t iz = pl.own_lo[2]; iz <= pl.own_hi[2]; ++iz)
        for (int64_t iy = pl.own_lo[1]; iy <= pl.own_hi[1]; ++iy) {
            const int64_t g0 = pl.own_lo[0] + NX * (iy + NY * iz);
            memcpy(local + l, global + g0, sizeof(double) * pl.own_n[0]);
            l += pl.own_n[0];
        }
}
static void scatter_owned(const Plan &pl, const double *local, double *global) {
    const int64_t NX = pl.mesh.NX(), NY = pl.mesh.NY();
    int64_t l = 0;
    for (int64_t iz = pl.own_lo[2]; iz <= pl.own_hi[2]; ++iz)
        for (int64_t iy = pl.own_lo[1]; iy <= pl.own_hi[1]; ++iy) {
            const int64_t g0 = pl.own_lo[0] + NX * (iy + NY * iz);
            memcpy(global + g0, local + l, sizeof(double) * pl.own_n[0]);
            l += pl.own_n[0];
        }
}
// owned-row-order values -> extended-box vector (halo columns left 0)
static void rows_to_cols(const Plan &pl, const double *rowv, double *colv) {
    int64_t l = 0;
    for (int64_t lz = 0; lz < pl.own_n[2]; ++lz)
        for (int64_t ly = 0; ly < pl.own_n[1]; ++ly) {
            const int64_t c0 = pl.off[0] + pl.ext_n[0] * ((ly + pl.off[1]) +
                                                          pl.ext_n[1] * (lz + pl.off[2]));
            memcpy(colv + c0, rowv + l, sizeof(double) * pl.own_n[0]);
            l += pl.own_n[0];
        }
}

// ----------------------------------------------------------------------------------------
// SpMV through the ABI
// ----------------------------------------------------------------------------------------

extern "C" int minife_spmv(minife_ctx *c, const double *x, double *y) {
    NvtxRange nvtx_("minife_spmv");
    if (!c || !x || !y) return MINIFE_EINVAL;
    if (!c->assembled) return MINIFE_ESTATE;
    const bool global_io = c->mode != MINIFE_MODE_RANK;
    std::vector<double> tmp, colv;
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        if (!p.d_xin) {
            TRY(alloc_colvec(c, p, &p.d_xin));
            TRY(dalloc(c, p, &p.d_yout, p.rows));
        }
        const double *src = x;
        if (global_io && !(c->parts.size() == 1 && p.ncols == p.rows)) {
            tmp.resize(p.rows);
            gather_owned(p.plan, x, tmp.data());
            src = tmp.data();
        }
        // stream-ordered with the SpMV below (a pageable cudaMemcpy may return before its DMA
        // lands, and the legacy stream is not ordered with the non-blocking ctx streams)
        cudaStream_t s = launch_stream(c, p);
        if (p.ncols == p.rows) {
            CUDA_TRY(c, cudaMemcpyAsync(p.d_xin, src, sizeof(double) * p.rows,
                                        cudaMemcpyHostToDevice, s));
        } else {
            colv.assign(p.ncols, 0.0);
            rows_to_cols(p.plan, src, colv.data());
            CUDA_TRY(c, cudaMemcpyAsync(p.d_xin, colv.data(), sizeof(double) * p.ncols,
                                        cudaMemcpyHostToDevice, s));
        }
        CUDA_TRY(c, cudaStreamSynchronize(s));     // tmp/colv are reused by the next part
    }
    TRY(enqueue_halo(c, [](Part &p) { return p.d_xin; }));
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        LAUNCH(c, launch_spmv(spmv_args(c, p, p.d_xin, p.d_yout, false), false, p.grid_spmv,
                                launch_stream(c, p)));
    }
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        CUDA_TRY(c, cudaStreamSynchronize(launch_stream(c, p)));
        if (global_io && !(c->parts.size() == 1 && p.ncols == p.rows)) {
            tmp.resize(p.rows);
            CUDA_TRY(c, cudaMemcpy(tmp.data(), p.d_yout, sizeof(double) * p.rows,
                                   cudaMemcpyDeviceToHost));
            scatter_owned(p.plan, tmp.data(), y);
        } else {
            CUDA_TRY(c, cudaMemcpy(y, p.d_yout, sizeof(double) * p.rows, cudaMemcpyDeviceToHost));
        }
    }
    return MINIFE_OK;
}

extern "C" int minife_spmv_device(minife_ctx *c, const double *d_x, double *d_y, void *stream) {
    if (!c || !d_x || !d_y) return MINIFE_EINVAL;
    if (c->mode != MINIFE_MODE_SINGLE || !c->assembled) return MINIFE_ESTATE;
    Part &p = c->parts[0];
    DevGuard g(p.dev);
    cudaStream_t s = stream ? (cudaStream_t)stream : stream_of(c, p);
    LAUNCH(c, launch_spmv(spmv_args(c, p, d_x, d_y, false), false, p.grid_spmv, s));
    return MINIFE_OK;
}

// ----------------------------------------------------------------------------------------
// getters
// ----------------------------------------------------------------------------------------

static void fill_part_info(const Plan &pl, int dev, int64_t entries, minife_part_info *o) {
    memset(o, 0, sizeof *o);
    o->rank = pl.rank;
    o->world = pl.world;
    for (int k = 0; k < 3; ++k) {
        o->box[k] = pl.boxes[pl.rank].lo[k];
        o->box[3 + k] = pl.boxes[pl.rank].hi[k];
        o->own[k] = pl.own_lo[k];
        o->own[3 + k] = pl.own_hi[k];
    }
    o->n_neighbors = (int32_t)pl.nbr.size();
    o->device = dev;
    o->rows = pl.n_owned;
    o->externals = pl.n_ext;
    o->nnz = pl.local_nnz();
    o->slices = (pl.n_owned + 31) / 32;
    o->sell_entries = entries;
    o->send_total = (int64_t)pl.send_idx.size();
    std::vector<int32_t> order;
    o->interior_slices = pl.slice_order(order);
}

extern "C" int minife_get_info(const minife_ctx *c, minife_info *o) {
    if (!c || !o) return MINIFE_EINVAL;
    memset(o, 0, sizeof *o);
    o->nx = c->mesh.nx;
    o->ny = c->mesh.ny;
    o->nz = c->mesh.nz;
    o->mode = c->mode;
    o->nparts = (int)c->parts.size();
    o->rank = c->rank;
    o->world = c->world;
    o->assembled = c->assembled;
    o->rows = c->mesh.rows();
    o->nnz = c->mesh.nnz();
    o->format = c->fmt;
    o->kernel_launches = c->kernel_launches + c->enq_kernels;
    o->comm = devcomm(c) ? 2 : ((c->world > 1 && c->mode != MINIFE_MODE_VIRTUAL) ? 1 : 0);
    for (auto &p : c->parts) {
        o->local_rows += p.rows;
        o->local_nnz += p.nnz;
        o->local_nns += p.nns;
        o->max_part_rows = std::max(o->max_part_rows, p.rows);
        o->max_part_nnz = std::max(o->max_part_nnz, p.nnz);
        o->max_part_externals = std::max(o->max_part_externals, p.plan.n_ext);
        o->sell_entries += p.entries;
        o->device_bytes += (int64_t)p.bytes;
    }
    return MINIFE_OK;
}

// ----------------------------------------------------------------------------------------
// verification and report data: rooted collectives (§3.2: data only process 0
// needs travels by Reduce / Gather, not Allreduce / Allgather)
// ----------------------------------------------------------------------------------------

extern "C" int minife_verify(minife_ctx *c, int64_t n, const int64_t *gids, int nterms,
                             double *u_fe, double *u_exact, double *max_abs_err) {
    NvtxRange nvtx_("minife_verify");
    if (!c || n < 0 || n > (1 << 24) || nterms < 1 || nterms > 4096 || !max_abs_err ||
        (n && (!gids || !u_fe || !u_exact)))
        return MINIFE_EINVAL;
    if (!c->solved) return MINIFE_ESTATE;
    const Mesh &m = c->mesh;
    for (int64_t i = 0; i < n; ++i)
        if (gids[i] < 0 || gids[i] >= m.rows()) return MINIFE_EINVAL;
    const bool use_nccl = c->mode == MINIFE_MODE_RANK || (c->mode == MINIFE_MODE_MULTI && c->world > 1);
    const bool root = c->mode != MINIFE_MODE_RANK || c->rank == 0;
    std::vector<double> total(2 * n, 0.0);
    double max_err = 0.0;
    std::vector<double *> bufs(c->parts.size(), nullptr);
    int st = MINIFE_OK;
    for (size_t q = 0; q < c->parts.size() && st == MINIFE_OK; ++q) {
        Part &p = c->parts[q];
        DevGuard g(p.dev);
        cudaStream_t s = launch_stream(c, p);
        std::vector<int64_t> lrow;
        std::vector<int32_t> ijk, slot;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t gid = gids[i];
            const int64_t ix = gid % m.NX(), iy = (gid / m.NX()) % m.NY(), iz = gid / (m.NX() * m.NY());
            if (!p.plan.owns(ix, iy, iz)) continue;
            lrow.push_back(p.plan.owned_local(ix, iy, iz));
            ijk.insert(ijk.end(), {(int32_t)ix, (int32_t)iy, (int32_t)iz});
            slot.push_back((int32_t)i);
        }
        const int k = (int)lrow.size();
        // one device block: [2n + 1 doubles out | k rows | 3k ijk | k slots]
        const size_t bytes = 8 * (2 * (size_t)n + 1) + 8 * (size_t)k + 4 * (size_t)(4 * k) + 16;
        char *blk = nullptr;
        CUDA_TRY(c, cudaMalloc((void **)&blk, bytes));
        bufs[q] = (double *)blk;
        double *out = (double *)blk;
        int64_t *d_row = (int64_t *)(blk + 8 * (2 * (size_t)n + 1));
        int32_t *d_ijk = (int32_t *)(d_row + k);
        int32_t *d_slot = d_ijk + 3 * k;
        cudaError_t e = cudaMemsetAsync(out, 0, 8 * (2 * (size_t)n + 1), s);
        if (e == cudaSuccess && k) e = cudaMemcpyAsync(d_row, lrow.data(), 8 * (size_t)k, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess && k) e = cudaMemcpyAsync(d_ijk, ijk.data(), 12 * (size_t)k, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess && k) e = cudaMemcpyAsync(d_slot, slot.data(), 4 * (size_t)k, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess && k) {
            e = launch_verify(p.d_x, m.nx, m.ny, m.nz, d_row, d_ijk, d_slot, k, nterms, out, s);
            if (e == cudaSuccess) ++c->enq_kernels;
        }
        // this part's largest |u_fe - u_exact| over its own probes -> word 2n of its block
        std::vector<double> mine(2 * n);
        if (e == cudaSuccess) e = cudaMemcpyAsync(mine.data(), out, 16 * (size_t)n, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        double local_max = 0.0;
        for (int j = 0; j < k; ++j)
            local_max = std::max(local_max, std::fabs(mine[2 * slot[j]] - mine[2 * slot[j] + 1]));
        if (e == cudaSuccess) e = cudaMemcpy(out + 2 * n, &local_max, 8, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            set_err(c, "verify: %s", cudaGetErrorString(e));
            st = MINIFE_ECUDA;
        }
        if (!use_nccl) {                 // one process, device-local parts: add on the host
            for (int j = 0; j < k; ++j) {
                total[2 * slot[j]] = mine[2 * slot[j]];
                total[2 * slot[j] + 1] = mine[2 * slot[j] + 1];
            }
            max_err = std::max(max_err, local_max);
        }
    }
    if (st == MINIFE_OK && use_nccl) {
        // every probe has exactly one owner and zeros elsewhere: the SUM reduce to rank 0 is
        // exact; the largest error by a MAX reduce of one word (rooted)
        ncclResult_t r = nccl()->GroupStart();
        for (size_t q = 0; q < c->parts.size() && r == ncclSuccess; ++q) {
            Part &p = c->parts[q];
            r = nccl()->Reduce(bufs[q], bufs[q], 2 * (size_t)n, ncclFloat64, ncclSum, 0, p.comm,
                               launch_stream(c, p));
            if (r == ncclSuccess)
                r = nccl()->Reduce(bufs[q] + 2 * n, bufs[q] + 2 * n, 1, ncclFloat64, ncclMax, 0,
                                   p.comm, launch_stream(c, p));
        }
        ncclResult_t r2 = nccl()->GroupEnd();
        if (r == ncclSuccess) r = r2;
        if (r != ncclSuccess) {
            set_err(c, "verify reduce: %s", nccl()->GetErrorString(r));
            st = MINIFE_ENCCL;
        }
        if (st == MINIFE_OK && root) {
            Part &p = c->parts[0];
            DevGuard g(p.dev);
            if (cudaStreamSynchronize(launch_stream(c, p)) != cudaSuccess ||
                cudaMemcpy(total.data(), bufs[0], 16 * (size_t)n, cudaMemcpyDeviceToHost) != cudaSuccess ||
                cudaMemcpy(&max_err, bufs[0] + 2 * n, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
                st = MINIFE_ECUDA;
        }
        for (auto &p : c->parts) {
            DevGuard g(p.dev);
            if (cudaStreamSynchronize(launch_stream(c, p)) != cudaSuccess) st = MINIFE_ECUDA;
        }
    }
    for (size_t q = 0; q < c->parts.size(); ++q) {
        DevGuard g(c->parts[q].dev);
        if (bufs[q]) cudaFree(bufs[q]);
    }
    if (st != MINIFE_OK || !root) return st;
    for (int64_t i = 0; i < n; ++i) {
        u_fe[i] = total[2 * i];
        u_exact[i] = total[2 * i + 1];
    }
    *max_abs_err = max_err;
    return MINIFE_OK;
}

extern "C" int minife_gather_times(minife_ctx *c, double *per_rank) {
    if (!c || !per_rank) return MINIFE_EINVAL;
    if (c->mode != MINIFE_MODE_RANK) {
        for (size_t q = 0; q < c->parts.size(); ++q) {
            per_rank[2 * q] = c->parts[q].t_asm_ms;
            per_rank[2 * q + 1] = c->parts[q].t_solve_ms;
        }
        return MINIFE_OK;
    }
    // rooted Gather (Allgather -> Gather): rank r sends its two numbers to rank 0 only
    Part &p = c->parts[0];
    DevGuard g(p.dev);
    cudaStream_t s = launch_stream(c, p);
    double *d = nullptr;
    const size_t words = 2 * (size_t)c->world;
    CUDA_TRY(c, cudaMalloc((void **)&d, 8 * words));
    const double mine[2] = {p.t_asm_ms, p.t_solve_ms};
    int st = MINIFE_OK;
    cudaError_t e = cudaMemcpyAsync(d + 2 * c->rank, mine, 16, cudaMemcpyHostToDevice, s);
    ncclResult_t r = ncclSuccess;
    if (e == cudaSuccess) {
        r = nccl()->GroupStart();
        if (c->rank == 0) {
            for (int q = 1; q < c->world && r == ncclSuccess; ++q)
                r = nccl()->Recv(d + 2 * q, 2, ncclFloat64, q, p.comm, s);
        } else if (r == ncclSuccess) {
            r = nccl()->Send(d + 2 * c->rank, 2, ncclFloat64, 0, p.comm, s);
        }
        ncclResult_t r2 = nccl()->GroupEnd();
        if (r == ncclSuccess) r = r2;
    }
    if (e == cudaSuccess && r == ncclSuccess && c->rank == 0)
        e = cudaMemcpyAsync(per_rank, d, 8 * words, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = MINIFE_ECUDA;
    if (r != ncclSuccess) {
        set_err(c, "gather: %s", nccl()->GetErrorString(r));
        st = MINIFE_ENCCL;
    }
    cudaFree(d);
    return st;
}

extern "C" int minife_get_timings(const minife_ctx *c, double *assemble_ms, double *solve_ms) {
    if (!c || !assemble_ms || !solve_ms) return MINIFE_EINVAL;
    *assemble_ms = c->last_asm_ms;
    *solve_ms = c->last_solve_ms;
    return MINIFE_OK;
}

extern "C" int minife_get_part_info(const minife_ctx *c, int part, minife_part_info *o) {
    if (!c || !o || part < 0 || part >= (int)c->parts.size()) return MINIFE_EINVAL;
    const Part &p = c->parts[part];
    fill_part_info(p.plan, p.dev, p.entries, o);
    return MINIFE_OK;
}

// rows [r0, r0+n) of one part -> (extended column, value) lists via the device extractor
static int extract_part_rows(minife_ctx *c, Part &p, const std::vector<int64_t> &loc,
                             std::vector<int32_t> &oc, std::vector<double> &ov,
                             std::vector<int32_t> &ol) {
    DevGuard g(p.dev);
    const int64_t k = (int64_t)loc.size();
    oc.assign(27 * k, 0);
    ov.assign(27 * k, 0.0);
    ol.assign(k, 0);
    if (!k) return MINIFE_OK;
    const int64_t chunk = 1 << 22;
    int64_t *d_rows = nullptr;
    int32_t *d_oc = nullptr, *d_ol = nullptr;
    double *d_ov = nullptr;
    const int64_t cap = std::min(k, chunk);
    CUDA_TRY(c, cudaMalloc((void **)&d_rows, 8 * cap));
    CUDA_TRY(c, cudaMalloc((void **)&d_oc, 4 * 27 * cap));
    CUDA_TRY(c, cudaMalloc((void **)&d_ov, 8 * 27 * cap));
    CUDA_TRY(c, cudaMalloc((void **)&d_ol, 4 * cap));
    int st = MINIFE_OK;
    for (int64_t b = 0; b < k && st == MINIFE_OK; b += chunk) {
        const int64_t n = std::min(chunk, k - b);
        cudaError_t e = cudaMemcpyAsync(d_rows, loc.data() + b, 8 * n, cudaMemcpyHostToDevice,
                                        p.stream);
        if (e == cudaSuccess)
            e = launch_extract_rows(matrix_of(c, p), geom_of(c, p), d_rows, n, d_oc, d_ov, d_ol,
                                    p.stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(p.stream);
        if (e == cudaSuccess)
            e = cudaMemcpy(oc.data() + 27 * b, d_oc, 4 * 27 * n, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess)
            e = cudaMemcpy(ov.data() + 27 * b, d_ov, 8 * 27 * n, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(ol.data() + b, d_ol, 4 * n, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            set_err(c, "extract rows: %s", cudaGetErrorString(e));
            st = MINIFE_ECUDA;
        }
    }
    cudaFree(d_rows);
    cudaFree(d_oc);
    cudaFree(d_ov);
    cudaFree(d_ol);
    return st;
}

extern "C" int minife_export_csr(minife_ctx *c, int64_t *row_ptr, int64_t *col, double *val) {
    if (!c || !row_ptr || !col || !val) return MINIFE_EINVAL;
    if (!c->assembled) return MINIFE_ESTATE;
    const Mesh &m = c->mesh;
    const bool local = c->mode == MINIFE_MODE_RANK;
    // row pointer from the closed-form row lengths (global id order, or owned rows)
    row_ptr[0] = 0;
    if (local) {
        const Plan &pl = c->parts[0].plan;
        for (int64_t r = 0; r < c->parts[0].rows; ++r) {
            const int64_t g = gid_of_row(pl, r);
            const int64_t ix = g % m.NX(), iy = (g / m.NX()) % m.NY(), iz = g / (m.NX() * m.NY());
            const int len = ((ix == 0 || ix == m.nx) ? 2 : 3) * ((iy == 0 || iy == m.ny) ? 2 : 3) *
                            ((iz == 0 || iz == m.nz) ? 2 : 3);
            row_ptr[r + 1] = row_ptr[r] + len;
        }
    } else {
        int64_t g = 0;
        for (int64_t iz = 0; iz < m.NZ(); ++iz)
            for (int64_t iy = 0; iy < m.NY(); ++iy)
                for (int64_t ix = 0; ix < m.NX(); ++ix, ++g) {
                    const int len = ((ix == 0 || ix == m.nx) ? 2 : 3) *
                                    ((iy == 0 || iy == m.ny) ? 2 : 3) *
                                    ((iz == 0 || iz == m.nz) ? 2 : 3);
                    row_ptr[g + 1] = row_ptr[g] + len;
                }
    }
    for (auto &p : c->parts) {
        std::vector<int64_t> loc(p.rows);
        for (int64_t r = 0; r < p.rows; ++r) loc[r] = r;
        std::vector<int32_t> oc, ol;
        std::vector<double> ov;
        TRY(extract_part_rows(c, p, loc, oc, ov, ol));
        for (int64_t r = 0; r < p.rows; ++r) {
            const int64_t out_row = local ? r : gid_of_row(p.plan, r);
            int64_t o = row_ptr[out_row];
            if (row_ptr[out_row + 1] - o != ol[r]) {
                set_err(c, "row %lld: device length %d != closed form", (long long)out_row, ol[r]);
                return MINIFE_ESTATE;
            }
            for (int e = 0; e < ol[r]; ++e) {
                col[o] = p.plan.col_to_gid(oc[27 * r + e]);
                val[o] = ov[27 * r + e];
                ++o;
            }
        }
    }
    return MINIFE_OK;
}

extern "C" int minife_export_rows(minife_ctx *c, int64_t n, const int64_t *gids, int64_t *cols,
                                  double *vals, int32_t *lens) {
    if (!c || n < 0 || (n && (!gids || !cols || !vals || !lens))) return MINIFE_EINVAL;
    if (!c->assembled) return MINIFE_ESTATE;
    const Mesh &m = c->mesh;
    for (int64_t i = 0; i < n; ++i) lens[i] = -1;
    for (auto &p : c->parts) {
        std::vector<int64_t> loc, which;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t gid = gids[i];
            if (gid < 0 || gid >= m.rows()) continue;
            const int64_t ix = gid % m.NX(), iy = (gid / m.NX()) % m.NY(),
                          iz = gid / (m.NX() * m.NY());
            if (!p.plan.owns(ix, iy, iz)) continue;
            loc.push_back(p.plan.owned_local(ix, iy, iz));
            which.push_back(i);
        }
        std::vector<int32_t> oc, ol;
        std::vector<double> ov;
        TRY(extract_part_rows(c, p, loc, oc, ov, ol));
        for (size_t j = 0; j < loc.size(); ++j) {
            const int64_t i = which[j];
            lens[i] = ol[j];
            for (int e = 0; e < ol[j]; ++e) {
                cols[27 * i + e] = p.plan.col_to_gid(oc[27 * j + e]);
                vals[27 * i + e] = ov[27 * j + e];
            }
        }
    }
    return MINIFE_OK;
}

static int get_vec(minife_ctx *c, double *out, double *Part::*member) {
    std::vector<double> tmp;
    for (auto &p : c->parts) {
        DevGuard g(p.dev);
        CUDA_TRY(c, cudaStreamSynchronize(launch_stream(c, p)));
        if (c->mode == MINIFE_MODE_RANK || (c->parts.size() == 1 && p.ncols == p.rows)) {
            // rows already in output order: copy straight into the caller's buffer
            CUDA_TRY(c, cudaMemcpy(out, p.*member, 8 * p.rows, cudaMemcpyDeviceToHost));
        } else {
            tmp.resize(p.rows);
            CUDA_TRY(c, cudaMemcpy(tmp.data(), p.*member, 8 * p.rows, cudaMemcpyDeviceToHost));
            scatter_owned(p.plan, tmp.data(), out);
        }
    }
    return MINIFE_OK;
}

extern "C" int minife_get_rhs(minife_ctx *c, double *b) {
    if (!c || !b) return MINIFE_EINVAL;
    if (!c->assembled) return MINIFE_ESTATE;
    return get_vec(c, b, &Part::d_b);
}

extern "C" int minife_get_solution(minife_ctx *c, double *x) {
    if (!c || !x) return MINIFE_EINVAL;
    if (!c->solved) return MINIFE_ESTATE;
    return get_vec(c, x, &Part::d_x);
}

extern "C" int minife_get_history(minife_ctx *c, double *h, int cap, int *n) {
    if (!c || !h || !n) return MINIFE_EINVAL;
    if (!c->solved) return MINIFE_ESTATE;
    const int cnt = c->last_iters + 1;
    *n = cnt;
    if (cap < cnt) return MINIFE_EINVAL;
    Part &p = c->parts[0];
    DevGuard g(p.dev);
    CUDA_TRY(c, cudaMemcpy(h, p.d_hist, 8 * cnt, cudaMemcpyDeviceToHost));
    return MINIFE_OK;
}

extern "C" int minife_get_owned_ids(const minife_ctx *c, int64_t *gids) {
    if (!c || !gids) return MINIFE_EINVAL;
    int64_t o = 0;
    for (auto &p : c->parts)
        for (int64_t l = 0; l < p.rows; ++l) gids[o++] = gid_of_row(p.plan, l);
    return MINIFE_OK;
}

// ----------------------------------------------------------------------------------------
// host-only plan queries
// ----------------------------------------------------------------------------------------

extern "C" int minife_plan(int nx, int ny, int nz, int world, int rank, minife_part_info *out) {
    if (!out || validate_mesh(nx, ny, nz) != MINIFE_OK) return MINIFE_EINVAL;
    Plan pl;
    if (!build_plan(Mesh{nx, ny, nz}, world, rank, pl)) return MINIFE_EINVAL;
    // CRS-format SELL entries from the closed-form row lengths (max per 32-row slice)
    int64_t entries = 0;
    {
        const Mesh m{nx, ny, nz};
        int64_t r = 0, w = 0;
        for (int64_t iz = pl.own_lo[2]; iz <= pl.own_hi[2]; ++iz)
            for (int64_t iy = pl.own_lo[1]; iy <= pl.own_hi[1]; ++iy)
                for (int64_t ix = pl.own_lo[0]; ix <= pl.own_hi[0]; ++ix) {
                    const int len = ((ix == 0 || ix == m.nx) ? 2 : 3) *
                                    ((iy == 0 || iy == m.ny) ? 2 : 3) *
                                    ((iz == 0 || iz == m.nz) ? 2 : 3);
                    w = std::max<int64_t>(w, len);
                    if ((++r & 31) == 0) {
                        entries += 32 * w;
                        w = 0;
                    }
                }
        if (r & 31) entries += 32 * w;
    }
    fill_part_info(pl, -1, entries, out);
    return MINIFE_OK;
}

extern "C" int minife_plan_lists(int nx, int ny, int nz, int world, int rank, int64_t *ext_gids,
                                 int32_t *nbr, int64_t *recv_cnt, int64_t *send_cnt,
                                 int32_t *send_idx) {
    if (validate_mesh(nx, ny, nz) != MINIFE_OK) return MINIFE_EINVAL;
    Plan pl;
    if (!build_plan(Mesh{nx, ny, nz}, world, rank, pl)) return MINIFE_EINVAL;
    if (ext_gids) std::copy(pl.ext_gid.begin(), pl.ext_gid.end(), ext_gids);
    for (size_t k = 0; k < pl.nbr.size(); ++k) {
        if (nbr) nbr[k] = pl.nbr[k];
        if (recv_cnt) recv_cnt[k] = pl.recv_cnt[k];
        if (send_cnt) send_cnt[k] = pl.send_cnt[k];
    }
    if (send_idx) std::copy(pl.send_idx.begin(), pl.send_idx.end(), send_idx);
    return MINIFE_OK;
}
