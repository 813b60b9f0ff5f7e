// plan.h — host-side RCB partition, nodal ownership and halo plans (G15; P:29, P:44-48;
// S:61-100).  Pure integer C++, no CUDA.
#pragma once
#include <cstdint>
#include <vector>

namespace minife {

struct Mesh {
    int nx, ny, nz;                       // elements per axis (G1)
    int64_t NX() const { return nx + 1; }
    int64_t NY() const { return ny + 1; }
    int64_t NZ() const { return nz + 1; }
    int64_t rows() const { return NX() * NY() * NZ(); }
    // stored entries of the full 27-point pattern: prod(3N-2)
    int64_t nnz() const { return (3 * NX() - 2) * (3 * NY() - 2) * (3 * NZ() - 2); }
};

struct Box {
    int lo[3], hi[3];                     // element ranges [lo, hi)
};

// RCB: longest axis (ties x<y<z), ceil(p/2) ranks take the lower part, cut at
// lo + floor(len*ceil(p/2)/p).  Returns false if some leaf would hold fewer elements than
// ranks.
bool rcb(const Mesh &m, int p, std::vector<Box> &boxes);

// Local numbering:
//   rows    = owned nodes, owned-box order (= ascending global id);
//   columns = the EXTENDED box = owned box grown by one node per side, clipped to the domain,
//             in its own x-fastest order.  It holds exactly owned ∪ externals, and every
//             x-run of the 27-point stencil is a run of consecutive columns, also across rank
//             boundaries — what lets one int32 index per run (the paper's BCRS segment,
//             P:116-124) describe every row.
//   halo slots (externals) keep the S:99 order (owner rank, global id) for the wire; ext_pos
//             maps slot -> extended column.
struct Plan {
    Mesh mesh;
    int rank = 0, world = 1;
    std::vector<Box> boxes;               // all ranks' element boxes
    int own_lo[3], own_hi[3];             // owned node box, inclusive
    int64_t own_n[3];
    int ext_lo[3];                        // extended box origin (global node coords)
    int64_t ext_n[3];
    int off[3];                           // own_lo - ext_lo (0 or 1 per axis)
    int64_t n_owned = 0, n_ext = 0, n_cols = 0;
    std::vector<int64_t> ext_gid;         // slot order: (owner rank, global id)
    std::vector<int64_t> ext_pos;         // slot -> extended column
    std::vector<int> nbr;                 // neighbor ranks, ascending
    std::vector<int64_t> recv_off, recv_cnt;   // slots [recv_off, +cnt) come from nbr[k]
    std::vector<int64_t> send_off, send_cnt;   // send_idx[send_off, +cnt) go to nbr[k]
    std::vector<int32_t> send_idx;        // local owned row indices

    int64_t owned_local(int64_t ix, int64_t iy, int64_t iz) const {
        return (ix - own_lo[0]) + own_n[0] * ((iy - own_lo[1]) + own_n[1] * (iz - own_lo[2]));
    }
    int64_t ext_col(int64_t ix, int64_t iy, int64_t iz) const {
        return (ix - ext_lo[0]) + ext_n[0] * ((iy - ext_lo[1]) + ext_n[1] * (iz - ext_lo[2]));
    }
    int64_t row_to_col(int64_t l) const {
        const int64_t lx = l % own_n[0], ly = (l / own_n[0]) % own_n[1],
                      lz = l / (own_n[0] * own_n[1]);
        return (lx + off[0]) + ext_n[0] * ((ly + off[1]) + ext_n[1] * (lz + off[2]));
    }
    int64_t col_to_gid(int64_t c) const {
        const int64_t a = c % ext_n[0], b = (c / ext_n[0]) % ext_n[1], d = c / (ext_n[0] * ext_n[1]);
        return (ext_lo[0] + a) + mesh.NX() * ((ext_lo[1] + b) + mesh.NY() * (ext_lo[2] + d));
    }
    int64_t local_nns() const;            // segments (x-runs) of the local rows
    bool owns(int64_t ix, int64_t iy, int64_t iz) const {
        return ix >= own_lo[0] && ix <= own_hi[0] && iy >= own_lo[1] && iy <= own_hi[1] &&
               iz >= own_lo[2] && iz <= own_hi[2];
    }
    int64_t local_nnz() const;            // closed form over the owned box

    // Row l reads a halo column iff its node lies on a face of the owned box beyond which
    // the domain continues (the node across that face is owned by another rank).
    bool row_reads_halo(int64_t l) const {
        const int64_t lc[3] = {l % own_n[0], (l / own_n[0]) % own_n[1],
                               l / (own_n[0] * own_n[1])};
        const int n[3] = {mesh.nx, mesh.ny, mesh.nz};
        for (int k = 0; k < 3; ++k) {
            if (lc[k] == 0 && own_lo[k] > 0) return true;
            if (lc[k] == own_n[k] - 1 && own_hi[k] < n[k]) return true;
        }
        return false;
    }
    // SELL-32 slice storage order for halo/interior overlap: the slices none of
    // whose rows reads a halo column first (ascending), then the others (ascending).
    // order[storage position] = row slice; returns the number of interior slices.
    int64_t slice_order(std::vector<int32_t> &order) const;
};

// Owned node box of `rank` (S:97 lowest-rank rule; DESIGN §4 shows it is a box: the closed
// node box minus every lower face lying on an interior cut plane).
void owned_box(const Mesh &m, const std::vector<Box> &boxes, int rank, int lo[3], int hi[3]);

// owner(node) = lowest rank whose closed node box contains it.
int owner_of(const std::vector<Box> &boxes, int64_t ix, int64_t iy, int64_t iz);

// Full plan of `rank`: owned box, externals, neighbors and halo send/recv lists.
bool build_plan(const Mesh &m, int world, int rank, Plan &out);

}  // namespace minife
