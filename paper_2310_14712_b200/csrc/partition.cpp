// Slab decomposition for world > 1 ranks.
//
// The box is cut into slabs of whole element layers along the last axis (z in 3D, y in 2D,
// x in 1D), with boundaries placed by a cost-weighted prefix sum (explicit bytes of the
// non-empty cells of a layer + dense cut K_e bytes + the implicit-solve bytes of each c
// component, charged to the layer of its centroid).  Ownership:
//   * a d node belongs to the rank whose slab holds its lattice plane (the last rank also
//     owns the top boundary plane);
//   * a c node belongs to the owner of its c component = the rank whose slab holds the
//     component's centroid layer, so every component's implicit solve is rank-local and the
//     solve needs no collective (void-aware ownership).
// Every rank keeps the FULL lattice state (2 x 8 B per node; config 5: 4.2 GB of 180 GB) and
// computes on its REGION: its slab grown to cover the c elements of its own components, plus
// one element layer of margin.  It updates every d node of the region whose incident elements
// all lie in the region (redundantly near the region boundary — same arithmetic, same bits)
// and the c part of its own components.  After each step it receives, from their owners, the
// region's nodes it does not update itself (d nodes on the region boundary, c nodes of other
// ranks' components): one point-to-point exchange with each overlapping rank per step.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "sc_internal.h"

// layers [lo, hi) of the split axis that a lattice plane z touches (its incident elements)
static inline void incident_layers(int64_t z, int P, int N, int& l0, int& l1) {
  if (z % P == 0) {
    l0 = (int)(z / P) - 1;
    l1 = (int)(z / P);
  } else {
    l0 = l1 = (int)(z / P);
  }
  if (l0 < 0) l0 = l1;
  if (l1 >= N) l1 = l0;
}

bool region_computes_plane(const sc_ctx* c, int q, int64_t z) {
  int l0, l1;
  const int ax = c->g.dim - 1;
  incident_layers(z, c->g.p, c->g.N[ax], l0, l1);
  return l0 >= c->reg_lo[q] && l1 < c->reg_hi[q];
}

int plane_owner(const sc_ctx* c, int64_t z) {
  for (int q = 0; q + 1 < c->world; ++q)
    if (z < (int64_t)c->layer_lo[q + 1] * c->g.p) return q;
  return c->world - 1;
}

void plan_partition(sc_ctx* c, const std::vector<CompSpan>& comps, std::vector<int>& owner) {
  const GridP& g = c->g;
  const int W = c->world, ax = g.dim - 1, N = g.N[ax];
  owner.assign(comps.size(), 0);
  c->layer_lo.assign(W + 1, 0);
  c->reg_lo.assign(W, 0);
  c->reg_hi.assign(W, N);
  c->layer_lo[W] = N;
  if (W == 1) return;
  if (N < W) throw ScError(SC_ERR_CONFIG, "fewer element layers than ranks along the split axis");
  // cost per element layer (bytes per step)
  int64_t nd_per_cell = 1;
  for (int k = 0; k < g.dim; ++k) nd_per_cell *= g.p;
  const double nb = (double)c->nb;
  std::vector<double> cost(N, 0.0);
  int64_t per_layer = 1;
  for (int k = 0; k < ax; ++k) per_layer *= g.N[k];
  for (int64_t cl = 0; cl < c->n_cells; ++cl) {
    const int L = (int)(cl / per_layer);
    const int8_t k = c->cell_class[cl];
    if (k == 0) cost[L] += 24.0 * (double)nd_per_cell;
    else if (k == 1) cost[L] += 8.0 * nb * nb;
  }
  for (const CompSpan& s : comps) cost[std::min(N - 1, std::max(0, s.centroid))] += s.cost;
  std::vector<double> pre(N + 1, 0.0);
  for (int L = 0; L < N; ++L) pre[L + 1] = pre[L] + cost[L];
  for (int q = 1; q < W; ++q) {
    const double target = pre[N] * q / W;
    int L = (int)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
    L = std::max(L, c->layer_lo[q - 1] + 1);     // at least one layer per rank
    L = std::min(L, N - (W - q));
    c->layer_lo[q] = L;
  }
  for (size_t k = 0; k < comps.size(); ++k) {
    int q = 0;
    while (q + 1 < W && comps[k].centroid >= c->layer_lo[q + 1]) ++q;
    owner[k] = q;
  }
  // regions: the slab grown over the own components' c elements, plus one margin layer
  for (int q = 0; q < W; ++q) {
    int lo = c->layer_lo[q], hi = c->layer_lo[q + 1];
    for (size_t k = 0; k < comps.size(); ++k)
      if (owner[k] == q) {
        lo = std::min(lo, comps[k].lmin);
        hi = std::max(hi, comps[k].lmax + 1);
      }
    c->reg_lo[q] = std::max(0, lo - 1);
    c->reg_hi[q] = std::min(N, hi + 1);
  }
}

// Exchange lists of this rank (deterministic: every rank derives every list from the same
// global classification and plan, so the sender's list for q and q's list for the sender
// agree element by element).  clat: lattice indices of all c nodes (ascending); c_owner: the
// owner rank of each.
void build_exchange(sc_ctx* c, const std::vector<int>& c_owner, const std::vector<int64_t>& clat) {
  const GridP& g = c->g;
  const int W = c->world, me = c->rank, ax = g.dim - 1, P = g.p;
  int64_t plane = 1;
  for (int k = 0; k < ax; ++k) plane *= g.nl[k];
  auto c_owner_of = [&](int64_t L) {
    const auto it = std::lower_bound(clat.begin(), clat.end(), L);
    return c_owner[it - clat.begin()];
  };
  // nodes of rank `reg`'s region that rank `src` owns and `reg` does not update itself
  auto list = [&](int src, int reg, std::vector<int32_t>& out) {
    const int64_t z0 = (int64_t)c->reg_lo[reg] * P;
    const int64_t z1 = std::min<int64_t>((int64_t)c->reg_hi[reg] * P, g.nl[ax] - 1);
    for (int64_t z = z0; z <= z1; ++z) {
      const bool computed = region_computes_plane(c, reg, z);
      const bool src_plane = plane_owner(c, z) == src;
      for (int64_t L = z * plane; L < (z + 1) * plane; ++L) {
        const uint8_t t = c->ntype[L];
        if (!t) continue;
        if (t == 3 ? (c_owner_of(L) == src) : (src_plane && !computed)) out.push_back((int32_t)L);
      }
    }
  };
  std::vector<int32_t> xs, xr;
  c->xs_off.assign(W + 1, 0);
  c->xr_off.assign(W + 1, 0);
  for (int q = 0; q < W; ++q) {
    c->xs_off[q] = (int64_t)xs.size();
    c->xr_off[q] = (int64_t)xr.size();
    if (q == me) continue;
    list(me, q, xs);
    list(q, me, xr);
  }
  c->xs_off[W] = (int64_t)xs.size();
  c->xr_off[W] = (int64_t)xr.size();
  auto up = [&](int32_t** d, double** buf, const std::vector<int32_t>& v) {
    SC_CUDA(cudaMalloc(d, sizeof(int32_t) * std::max<size_t>(1, v.size())));
    SC_CUDA(cudaMalloc(buf, sizeof(double) * std::max<size_t>(1, v.size())));
    if (!v.empty()) SC_CUDA(cudaMemcpy(*d, v.data(), sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice));
  };
  up(&c->d_xs_idx, &c->d_xs_buf, xs);
  up(&c->d_xr_idx, &c->d_xr_buf, xr);
  // owned DOFs (sc_read)
  c->own_dofs.clear();
  std::vector<int32_t> own_lat;
  for (int64_t i = 0; i < c->n_dof; ++i) {
    const int64_t L = c->dof_lat[i];
    const int o = c->ntype[L] == 3 ? c_owner_of(L) : plane_owner(c, L / plane);
    if (o == me) {
      c->own_dofs.push_back((int32_t)i);
      own_lat.push_back((int32_t)L);
    }
  }
  SC_CUDA(cudaMalloc(&c->d_own_lat, sizeof(int32_t) * std::max<size_t>(1, own_lat.size())));
  SC_CUDA(cudaMalloc(&c->d_own_dof, sizeof(int32_t) * std::max<size_t>(1, own_lat.size())));
  if (!own_lat.empty()) {
    SC_CUDA(cudaMemcpy(c->d_own_lat, own_lat.data(), sizeof(int32_t) * own_lat.size(), cudaMemcpyHostToDevice));
    SC_CUDA(cudaMemcpy(c->d_own_dof, c->own_dofs.data(), sizeof(int32_t) * own_lat.size(),
                       cudaMemcpyHostToDevice));
  }
}
