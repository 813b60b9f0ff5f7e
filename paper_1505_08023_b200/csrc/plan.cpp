// plan.cpp — RCB partition, ownership, externals and halo plans (host, integer only).
// Readings: G15 (S:64 split rule), S:97 (lowest-rank ownership), S:82/S:99 (externals and
// their order), S:293-296 (HaloPlan: consistent send/recv lists).
#include "plan.h"

#include <algorithm>

namespace minife {

static bool rcb_rec(const Box &b, int r0, int p, std::vector<Box> &out) {
    int64_t elems = (int64_t)(b.hi[0] - b.lo[0]) * (b.hi[1] - b.lo[1]) * (b.hi[2] - b.lo[2]);
    if (elems < p) return false;
    if (p == 1) {
        out[r0] = b;
        return true;
    }
    int axis = 0;
    for (int k = 1; k < 3; ++k)
        if (b.hi[k] - b.lo[k] > b.hi[axis] - b.lo[axis]) axis = k;
    const int plo = (p + 1) / 2, phi = p / 2;
    const int len = b.hi[axis] - b.lo[axis];
    const int cut = b.lo[axis] + (int)(((int64_t)len * plo) / p);
    Box lower = b, upper = b;
    lower.hi[axis] = cut;
    upper.lo[axis] = cut;
    return rcb_rec(lower, r0, plo, out) && rcb_rec(upper, r0 + plo, phi, out);
}

bool rcb(const Mesh &m, int p, std::vector<Box> &boxes) {
    if (m.nx < 1 || m.ny < 1 || m.nz < 1 || p < 1) return false;
    boxes.assign(p, Box{});
    Box all{{0, 0, 0}, {m.nx, m.ny, m.nz}};
    return rcb_rec(all, 0, p, boxes);
}

int owner_of(const std::vector<Box> &boxes, int64_t ix, int64_t iy, int64_t iz) {
    const int64_t c[3] = {ix, iy, iz};
    for (size_t r = 0; r < boxes.size(); ++r) {
        bool in = true;
        for (int k = 0; k < 3; ++k)
            if (c[k] < boxes[r].lo[k] || c[k] > boxes[r].hi[k]) in = false;
        if (in) return (int)r;
    }
    return -1;
}

// Every cut plane is interior (0 < c < n), and at the split that separates two ranks the
// lower-coordinate side holds the lower ranks; so the nodes of `rank`'s closed box shared
// with a lower rank are exactly those on its lower faces with lo > 0, and every such face
// is fully covered by lower ranks.  Owned set = closed box minus those faces (a box).
void owned_box(const Mesh &m, const std::vector<Box> &boxes, int rank, int lo[3], int hi[3]) {
    (void)m;
    for (int k = 0; k < 3; ++k) {
        lo[k] = boxes[rank].lo[k] + (boxes[rank].lo[k] > 0 ? 1 : 0);
        hi[k] = boxes[rank].hi[k];
    }
}

int64_t Plan::local_nnz() const {
    const int n[3] = {mesh.nx, mesh.ny, mesh.nz};
    int64_t prod = 1;
    for (int k = 0; k < 3; ++k) {
        int64_t s = 0;
        for (int i = own_lo[k]; i <= own_hi[k]; ++i) s += (i == 0 || i == n[k]) ? 2 : 3;
        prod *= s;
    }
    return n_owned == 0 ? 0 : prod;
}

int64_t Plan::slice_order(std::vector<int32_t> &order) const {
    const int64_t ns = (n_owned + 31) / 32;
    std::vector<int32_t> inner, outer;
    for (int64_t s = 0; s < ns; ++s) {
        bool halo = false;
        for (int64_t l = 32 * s; l < 32 * s + 32 && l < n_owned && !halo; ++l)
            halo = row_reads_halo(l);
        (halo ? outer : inner).push_back((int32_t)s);
    }
    order = inner;
    order.insert(order.end(), outer.begin(), outer.end());
    return (int64_t)inner.size();
}

// x-runs per row = (#present y-neighbors) * (#present z-neighbors): 9 inside, fewer on y/z
// boundary planes; summed separably over the owned box.
int64_t Plan::local_nns() const {
    const int n[3] = {mesh.nx, mesh.ny, mesh.nz};
    int64_t prod = own_n[0];
    for (int k = 1; k < 3; ++k) {
        int64_t s = 0;
        for (int i = own_lo[k]; i <= own_hi[k]; ++i) s += (i == 0 || i == n[k]) ? 2 : 3;
        prod *= s;
    }
    return n_owned == 0 ? 0 : prod;
}

// externals of rank r in slot order (owner rank, global id), with their owners
static void externals_of(const Mesh &m, const std::vector<Box> &boxes, int r,
                         std::vector<int64_t> &gid, std::vector<int> &own) {
    int lo[3], hi[3];
    owned_box(m, boxes, r, lo, hi);
    const int64_t N[3] = {m.NX(), m.NY(), m.NZ()};
    int64_t slo[3], shi[3];
    for (int k = 0; k < 3; ++k) {
        slo[k] = std::max<int64_t>(lo[k] - 1, 0);
        shi[k] = std::min<int64_t>(hi[k] + 1, N[k] - 1);
    }
    std::vector<std::pair<int, int64_t>> ext;
    for (int64_t iz = slo[2]; iz <= shi[2]; ++iz)
        for (int64_t iy = slo[1]; iy <= shi[1]; ++iy)
            for (int64_t ix = slo[0]; ix <= shi[0]; ++ix) {
                if (ix >= lo[0] && ix <= hi[0] && iy >= lo[1] && iy <= hi[1] && iz >= lo[2] &&
                    iz <= hi[2])
                    continue;
                int o = owner_of(boxes, ix, iy, iz);
                ext.emplace_back(o, ix + N[0] * (iy + N[1] * iz));
            }
    std::stable_sort(ext.begin(), ext.end(),
                     [](const std::pair<int, int64_t> &a, const std::pair<int, int64_t> &b) {
                         return a.first < b.first;
                     });
    gid.resize(ext.size());
    own.resize(ext.size());
    for (size_t i = 0; i < ext.size(); ++i) {
        own[i] = ext[i].first;
        gid[i] = ext[i].second;
    }
}

bool build_plan(const Mesh &m, int world, int rank, Plan &P) {
    if (world < 1 || rank < 0 || rank >= world) return false;
    P = Plan{};
    P.mesh = m;
    P.rank = rank;
    P.world = world;
    if (!rcb(m, world, P.boxes)) return false;
    owned_box(m, P.boxes, rank, P.own_lo, P.own_hi);
    const int64_t Nn[3] = {m.NX(), m.NY(), m.NZ()};
    for (int k = 0; k < 3; ++k) {
        P.own_n[k] = (int64_t)P.own_hi[k] - P.own_lo[k] + 1;
        P.ext_lo[k] = P.own_lo[k] > 0 ? P.own_lo[k] - 1 : 0;
        const int64_t ext_hi = std::min<int64_t>(P.own_hi[k] + 1, Nn[k] - 1);
        P.ext_n[k] = ext_hi - P.ext_lo[k] + 1;
        P.off[k] = P.own_lo[k] - P.ext_lo[k];
    }
    P.n_owned = P.own_n[0] * P.own_n[1] * P.own_n[2];
    P.n_cols = P.ext_n[0] * P.ext_n[1] * P.ext_n[2];
    std::vector<int> owners;
    externals_of(m, P.boxes, rank, P.ext_gid, owners);
    P.n_ext = (int64_t)P.ext_gid.size();
    P.ext_pos.resize(P.n_ext);
    for (int64_t i = 0; i < P.n_ext; ++i) {
        const int64_t g = P.ext_gid[i];
        P.ext_pos[i] = P.ext_col(g % Nn[0], (g / Nn[0]) % Nn[1], g / (Nn[0] * Nn[1]));
    }
    if (P.n_owned + P.n_ext != P.n_cols) return false;   // extended box == owned ∪ externals
    for (size_t i = 0; i < owners.size(); ++i) {
        if (P.nbr.empty() || P.nbr.back() != owners[i]) {
            P.nbr.push_back(owners[i]);
            P.recv_off.push_back((int64_t)i);
            P.recv_cnt.push_back(0);
        }
        P.recv_cnt.back()++;
    }
    // send lists: what each neighbor s expects from us, in s's slot order
    const int64_t NX = m.NX(), NY = m.NY();
    for (size_t k = 0; k < P.nbr.size(); ++k) {
        std::vector<int64_t> g;
        std::vector<int> o;
        externals_of(m, P.boxes, P.nbr[k], g, o);
        P.send_off.push_back((int64_t)P.send_idx.size());
        int64_t cnt = 0;
        for (size_t i = 0; i < g.size(); ++i) {
            if (o[i] != rank) continue;
            int64_t ix = g[i] % NX, iy = (g[i] / NX) % NY, iz = g[i] / (NX * NY);
            P.send_idx.push_back((int32_t)P.owned_local(ix, iy, iz));
            ++cnt;
        }
        P.send_cnt.push_back(cnt);
    }
    return true;
}

}  // namespace minife
