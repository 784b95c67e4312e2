// C ABI entry points of libsc (include/sc.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sc_internal.h"

static thread_local std::string g_setup_err;

static sc_status fail(sc_ctx* c, const ScError& e) {
  if (c) c->err = e.msg;
  else g_setup_err = e.msg;
  return e.st;
}

// SC_TRACE=path: dump the last solve launch's item timeline (debug instrumentation)
static void dump_trace(sc_ctx* c) {
  const char* path = getenv("SC_TRACE");
  if (!path || !c->d_trace || c->n_items == 0) return;
  std::vector<unsigned long long> t(5 * (size_t)c->n_items);
  if (cudaMemcpy(t.data(), c->d_trace, sizeof(unsigned long long) * t.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
    return;
  FILE* f = fopen(path, "wb");
  if (!f) return;
  const int32_t hdr[2] = {c->n_items, c->n_sn};
  fwrite(hdr, sizeof(int32_t), 2, f);
  fwrite(c->h_items.data(), sizeof(int32_t), c->h_items.size(), f);
  fwrite(t.data(), sizeof(unsigned long long), t.size(), f);
  std::vector<int32_t> wr(3 * (size_t)c->n_sn);
  cudaMemcpy(wr.data(), c->d_sn_w, sizeof(int32_t) * c->n_sn, cudaMemcpyDeviceToHost);
  cudaMemcpy(wr.data() + c->n_sn, c->d_sn_r, sizeof(int32_t) * c->n_sn, cudaMemcpyDeviceToHost);
  cudaMemcpy(wr.data() + 2 * c->n_sn, c->d_parent, sizeof(int32_t) * c->n_sn, cudaMemcpyDeviceToHost);
  fwrite(wr.data(), sizeof(int32_t), wr.size(), f);
  fclose(f);
}

static void free_ctx(sc_ctx* c) {
  if (!c) return;
  int cur = -1;
  cudaGetDevice(&cur);
  cudaSetDevice(c->device);
  dump_trace(c);
  try {
    nccl_destroy(c);
  } catch (const ScError&) {
  }
  destroy_graphs(c);
  void* ptrs[] = {c->d_voids, c->d_u[0], c->d_u[1], c->d_ntype, c->d_cell_class, c->d_dof_lat, c->d_out,
                  c->d_ft, c->d_step, c->d_flag, c->d_irr_lat, c->d_irr_invm, c->d_irr_fx, c->d_load_lat, c->d_load_fxm, c->d_Kref,
                  c->d_c_lat, c->d_vc, c->d_ac, c->d_fxc, c->d_b, c->d_q, c->d_x, c->d_U,
                  c->d_celem_cell, c->d_celem_kidx, c->d_celem_cidx, c->d_celem_cut_ids, c->d_celem_ref_ids,
                  c->d_Kcut, c->d_Kpk, c->d_cut_dt, c->d_Y, c->d_rhs_ptr,
                  c->d_rhs_idx, c->d_sn_c0, c->d_sn_w, c->d_sn_r, c->d_sn_aoff, c->d_sn_roff,
                  c->d_sn_uoff, c->d_sn_goff, c->d_R, c->d_gptr, c->d_gidx, c->d_items, c->fS.A,
                  c->fM.A, c->fS.d, c->fM.d, c->d_tmp, c->d_nitem, c->d_chptr, c->d_chidx, c->d_parent, c->d_solve_cnt,
                  c->d_part, c->d_trace, c->d_near_tiles, c->d_qmeta, c->d_far_tiles, c->d_xs_idx, c->d_xr_idx,
                  c->d_xs_buf, c->d_xr_buf, c->d_stage, c->d_vlat, c->d_own_lat, c->d_own_dof, c->d_full, c->d_clean, c->d_rec_lat, c->d_rec_w,
                  c->d_rec_trace, c->d_mc, c->d_g2};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->s_hi) cudaStreamDestroy(c->s_hi);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->s_ref) cudaStreamDestroy(c->s_ref);
  if (c->ev_ref0) cudaEventDestroy(c->ev_ref0);
  if (c->ev_ref1) cudaEventDestroy(c->ev_ref1);
  if (cur >= 0) cudaSetDevice(cur);
  delete c;
}

static void validate(const sc_grid* grid, int32_t p, double alpha, const sc_geometry* geom, double dt,
                     const sc_source* src) {
  if (!grid || !geom) throw ScError(SC_ERR_CONFIG, "grid and geometry are required");
  if (grid->dim < 1 || grid->dim > 3) throw ScError(SC_ERR_CONFIG, "dim must be 1, 2 or 3");
  for (int k = 0; k < grid->dim; ++k) {
    if (grid->cells[k] < 1) throw ScError(SC_ERR_CONFIG, "cells must be >= 1");
    if (!(grid->hi[k] > grid->lo[k])) throw ScError(SC_ERR_CONFIG, "hi must exceed lo");
  }
  if (p < 1 || p > 8) throw ScError(SC_ERR_CONFIG, "p must be in [1, 8]");
  if (grid->dim == 3 && p > 6) throw ScError(SC_ERR_CONFIG, "3D supports p <= 6");
  if (!(alpha > 0.0) || !(alpha <= 1.0)) throw ScError(SC_ERR_CONFIG, "alpha must be in (0, 1]");
  if (!(dt > 0.0) || !std::isfinite(dt)) throw ScError(SC_ERR_CONFIG, "dt must be positive");
  if (geom->n_voids < 0 || geom->n_voids > SC_MAX_VOIDS || (geom->n_voids > 0 && !geom->voids))
    throw ScError(SC_ERR_CONFIG, "invalid void list");
  if (geom->tree_depth < 0 || geom->tree_depth > 12) throw ScError(SC_ERR_CONFIG, "tree_depth in [0, 12]");
  if (geom->lattice_s < 1 || geom->lattice_s > 16) throw ScError(SC_ERR_CONFIG, "lattice_s in [1, 16]");
  if (!(geom->rho > 0.0) || !(geom->c > 0.0)) throw ScError(SC_ERR_CONFIG, "rho and c must be positive");
  if (src && (src->kind < 0 || src->kind > 2)) throw ScError(SC_ERR_CONFIG, "source kind must be 0, 1 or 2");
  if (src && src->kind >= 1 && (src->n_t < 0 || (src->n_t > 0 && !src->f_t)))
    throw ScError(SC_ERR_CONFIG, "invalid source signal");
  for (int i = 0; i < geom->n_voids; ++i) {
    const sc_void& v = geom->voids[i];
    if (v.kind != SC_VOID_ELLIPSOID && v.kind != SC_VOID_HALFSPACE) throw ScError(SC_ERR_CONFIG, "void kind");
  }
  // empty-cell rule (reading C7): a cell is EMPTY iff none of its Gauss
  // points is physical.  That integer decision equals "eta < fill_eps" exactly when the smallest
  // nonzero fill ratio a cell can have - one physical Gauss point of the smallest weight on a
  // depth-D leaf, eta_min = (2^-D * w_min / 2)^dim - is >= fill_eps; deeper trees (or a larger
  // fill_eps) would make the two rules differ, so they are rejected instead of silently ignored.
  if (!(geom->fill_eps >= 0.0) || !(geom->fill_eps < 1.0)) throw ScError(SC_ERR_CONFIG, "fill_eps must be in [0, 1)");
  {
    std::vector<double> gx, gw;
    host_gauss(p + 1, gx, gw);
    double wmin = gw[0];
    for (double w : gw) wmin = std::min(wmin, w);
    const double eta_min = std::pow(std::ldexp(0.5 * wmin, -geom->tree_depth), grid->dim);
    if (eta_min < geom->fill_eps)
      throw ScError(SC_ERR_CONFIG, "fill_eps exceeds the smallest nonzero fill ratio of this tree_depth/p/dim "
                                   "(the empty rule 'no physical Gauss point' would differ from eta < fill_eps)");
  }
}

extern "C" sc_status sc_setup(const sc_grid* grid, int32_t p, double alpha, const sc_geometry* geom, double dt,
                              const sc_source* src, const double* u0, const double* v0, const sc_dist* dist,
                              sc_ctx** out) {
  if (!out) return SC_ERR_STATE;
  *out = nullptr;
  sc_ctx* c = nullptr;
  auto t0 = std::chrono::steady_clock::now();
  try {
    validate(grid, p, alpha, geom, dt, src);
    c = new sc_ctx();
    c->device = dist ? dist->device : -1;
    if (c->device < 0) SC_CUDA(cudaGetDevice(&c->device));
    SC_CUDA(cudaSetDevice(c->device));
    if (dist) {
      if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world)
        throw ScError(SC_ERR_CONFIG, "dist: need 0 <= rank < world");
      c->rank = dist->rank;
      c->world = dist->world;
    }
    if (dist && dist->cuda_stream) {
      c->stream = (cudaStream_t)dist->cuda_stream;
    } else {
      SC_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    GridP& g = c->g;
    g.dim = grid->dim;
    g.p = p;
    g.s = geom->lattice_s;
    g.depth = geom->tree_depth;
    g.ezl = 0;
    c->nb = 1;
    c->n_cells = 1;
    c->n_lat = 1;
    for (int k = 0; k < 3; ++k) {
      if (k < g.dim) {
        g.N[k] = grid->cells[k];
        g.lo[k] = grid->lo[k];
        g.hi[k] = grid->hi[k];
        g.h[k] = (grid->hi[k] - grid->lo[k]) / grid->cells[k];
        g.nl[k] = (int64_t)g.N[k] * p + 1;
        c->nb *= p + 1;
      } else {
        g.N[k] = 1;
        g.lo[k] = 0.0;
        g.hi[k] = 0.0;
        g.h[k] = 1.0;
        g.nl[k] = 1;
      }
      c->n_cells *= g.N[k];
      c->n_lat *= g.nl[k];
    }
    if (c->n_lat >= (1LL << 31)) throw ScError(SC_ERR_CONFIG, "lattice larger than 2^31 nodes");
    c->alpha = alpha;
    c->rho = geom->rho;
    c->c = geom->c;
    c->dt = dt;
    c->fill_eps = geom->fill_eps;
    if (geom->integrator < 0 || geom->integrator > 4) throw ScError(SC_ERR_CONFIG, "integrator must be 0..4");
    c->integrator = geom->integrator;
    if (c->integrator == 4) {
      if (geom->lf_m < 1 || geom->lf_m > 64) throw ScError(SC_ERR_CONFIG, "leap-frog: lf_m must be in [1, 64]");
      if (geom->lf_coupling != 0 && geom->lf_coupling != 1) throw ScError(SC_ERR_CONFIG, "leap-frog: lf_coupling 0 or 1");
      if (dist && dist->world > 1) throw ScError(SC_ERR_CONFIG, "leap-frog: one rank only");
      c->lf_m = geom->lf_m;
      c->lf_coupling = geom->lf_coupling;
    }
    for (int i = 0; i < geom->n_voids; ++i) {
      DVoid v;
      std::memset(&v, 0, sizeof(v));
      const sc_void& s = geom->voids[i];
      v.kind = s.kind;
      for (int k = 0; k < 3; ++k) {
        v.c[k] = s.c[k];
        v.n[k] = s.n[k];
      }
      for (int k = 0; k < 6; ++k) v.A[k] = s.A[k];
      v.b = s.b;
      c->voids.push_back(v);
    }
    if (src && (src->kind == 1 || src->kind == 2)) {
      c->src_kind = src->kind;
      for (int k = 0; k < 3; ++k) c->src_x[k] = src->x[k];
      if (src->kind == 2) {
        if (!(src->sigma > 0.0) || !std::isfinite(src->amp)) throw ScError(SC_ERR_CONFIG, "bell source: sigma > 0");
        c->src_sigma = src->sigma;
        c->src_amp = src->amp;
      }
    }
    // SC_SETUP_TIMES (diagnostics): setup phase times on stderr
    auto lap = [&, tl = std::chrono::steady_clock::now()](const char* what) mutable {
      const auto now = std::chrono::steady_clock::now();
      if (getenv("SC_SETUP_TIMES")) fprintf(stderr, "sc_setup %-22s %8.3f s\n", what, std::chrono::duration<double>(now - tl).count());
      tl = now;
    };
    host_reference(c);
    device_upload_reference(c);
    lap("reference");
    setup_device_geometry(c);
    lap("geometry+cut matrices");
    setup_factor(c, {});
    lap("factorisation");
    setup_step_structures(c);
    lap("step structures");
    // state buffers
    const size_t latb = sizeof(double) * c->n_lat;
    SC_CUDA(cudaMalloc(&c->d_u[0], latb));
    SC_CUDA(cudaMalloc(&c->d_u[1], latb));
    SC_CUDA(cudaMalloc(&c->d_step, sizeof(long long)));
    SC_CUDA(cudaMalloc(&c->d_flag, sizeof(int)));
    SC_CUDA(cudaMalloc(&c->d_dof_lat, sizeof(int64_t) * std::max<int64_t>(1, c->n_dof)));
    SC_CUDA(cudaMemcpy(c->d_dof_lat, c->dof_lat.data(), sizeof(int64_t) * c->n_dof, cudaMemcpyHostToDevice));
    SC_CUDA(cudaMalloc(&c->d_out, sizeof(double) * std::max<int64_t>(1, c->n_dof)));
    c->n_t = (src && (src->kind == 1 || src->kind == 2)) ? src->n_t : 0;
    SC_CUDA(cudaMalloc(&c->d_ft, sizeof(double) * std::max<int64_t>(1, c->n_t)));
    if (c->n_t) SC_CUDA(cudaMemcpy(c->d_ft, src->f_t, sizeof(double) * c->n_t, cudaMemcpyHostToDevice));
    // algorithmic bytes per step
    {
      const double nbd = (double)c->nb;
      // tensor-d nodes (the explicit launch, sc_profile 0): read u_n, u_{n-1}; write u_{n+1}
      const double ex = 24.0 * (double)(c->n_d - c->n_irr);
      // c-element products: each cut K_e once (packed lower triangle, else dense), w gathered
      // and Y written per element node
      const double kb = c->d_Kpk ? nbd * (nbd + 1.0) / 2.0 : nbd * nbd;
      const double ce = 8.0 * (double)c->n_cut * kb + 16.0 * (double)c->n_celem * nbd;
      // solve: forward streams every panel [D_s; G_s], backward G_s again; b, q, x vectors
      // and the update vectors U (written once, read once)
      const double so = 8.0 * (double)(c->nnz_factor + c->nnz_G) + 32.0 * (double)c->n_cl + 16.0 * (double)c->sum_r;
      c->bytes_explicit = ex;
      c->bytes_celem = ce;
      c->bytes_solve = so;
      c->bytes_per_step = ex + 24.0 * (double)c->n_irr + ce + so +
                          56.0 * (double)c->n_cl;   // r^c gather + corrector state (u, v, a, x)
    }
    if (u0) SC_CUDA(cudaMemcpy(c->d_out, u0, sizeof(double) * c->n_dof, cudaMemcpyHostToDevice));
    if (v0) {
      SC_CUDA(cudaMalloc(&c->d_stage, sizeof(double) * std::max<int64_t>(1, c->n_dof)));
      SC_CUDA(cudaMemcpy(c->d_stage, v0, sizeof(double) * c->n_dof, cudaMemcpyHostToDevice));
    }
    run_startup(c, u0 ? c->d_out : nullptr, v0 ? c->d_stage : nullptr);
    build_graphs(c);
    if (c->world > 1 && dist->nccl_unique_id) nccl_init(c, dist->nccl_unique_id);
    SC_CUDA(cudaStreamSynchronize(c->stream));
    c->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = c;
    return SC_OK;
  } catch (const ScError& e) {
    g_setup_err = e.msg;
    free_ctx(c);
    return e.st;
  } catch (const std::bad_alloc&) {
    g_setup_err = "host allocation failed";
    free_ctx(c);
    return SC_ERR_OOM;
  }
}

extern "C" sc_status sc_set_state(sc_ctx* c, const double* u0, const double* v0, int64_t len) {
  if (!c) return SC_ERR_STATE;
  if ((u0 || v0) && len != c->n_dof) {
    c->err = "sc_set_state: len must equal n_dof (" + std::to_string(c->n_dof) + ")";
    return SC_ERR_CONFIG;
  }
  try {
    SC_CUDA(cudaSetDevice(c->device));
    // staged through context-owned buffers (no per-call allocation): u0 -> d_out, v0 -> d_stage
    const size_t nbytes = sizeof(double) * c->n_dof;
    if (u0) SC_CUDA(cudaMemcpyAsync(c->d_out, u0, nbytes, cudaMemcpyHostToDevice, c->stream));
    if (v0) {
      if (!c->d_stage) SC_CUDA(cudaMalloc(&c->d_stage, sizeof(double) * std::max<int64_t>(1, c->n_dof)));
      SC_CUDA(cudaMemcpyAsync(c->d_stage, v0, nbytes, cudaMemcpyHostToDevice, c->stream));
    }
    run_startup(c, u0 ? c->d_out : nullptr, v0 ? c->d_stage : nullptr);
    return SC_OK;
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_step(sc_ctx* c, int64_t n) {
  if (!c) return SC_ERR_STATE;
  if (n < 0) {
    c->err = "n must be >= 0";
    return SC_ERR_CONFIG;
  }
  try {
    SC_CUDA(cudaSetDevice(c->device));
    if (n > 0) enqueue_far_prologue(c);
    for (int64_t i = 0; i < n; ++i) {
      SC_CUDA(cudaGraphLaunch(c->graph[c->cur], c->stream));   // world > 1: ends with the pack
      c->cur ^= 1;
      ++c->host_step;
      if (c->world > 1 && c->nccl_comm) {
        nccl_exchange(c);
        enqueue_unpack(c, c->d_u[c->cur], c->stream);
      }
    }
    return SC_OK;
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_sync(sc_ctx* c) {
  if (!c) return SC_ERR_STATE;
  try {
    SC_CUDA(cudaSetDevice(c->device));
    int flag = 0;
    SC_CUDA(cudaMemcpyAsync(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    SC_CUDA(cudaStreamSynchronize(c->stream));
    if (flag) {
      c->err = "non-finite value in the state (instability)";
      return SC_ERR_NUMERIC;
    }
    return SC_OK;
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_read(sc_ctx* c, double* u, int64_t len) {
  if (!c) return SC_ERR_STATE;
  if (!u || len < c->n_dof) {
    c->err = "output buffer too small";
    return SC_ERR_CONFIG;
  }
  try {
    SC_CUDA(cudaSetDevice(c->device));
    if (c->world > 1) {
      // every DOF is owned by exactly one rank: sum of the owned parts = the field
      if (!c->nccl_comm) {
        c->err = "world > 1 without NCCL (in-process ranks): use sc_read_owned on every rank";
        return SC_ERR_STATE;
      }
      SC_CUDA(cudaMemsetAsync(c->d_out, 0, sizeof(double) * c->n_dof, c->stream));
      gather_owned(c, c->d_u[c->cur], c->d_out);
      nccl_allreduce_sum(c, c->d_out, c->n_dof);
    } else {
      gather_dofs(c, c->d_u[c->cur], c->d_out);
    }
    SC_CUDA(cudaMemcpyAsync(u, c->d_out, sizeof(double) * c->n_dof, cudaMemcpyDeviceToHost, c->stream));
    return sc_sync(c);
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_read_owned(sc_ctx* c, double* u, int64_t len) {
  if (!c) return SC_ERR_STATE;
  if (!u || len < c->n_dof) {
    c->err = "output buffer too small";
    return SC_ERR_CONFIG;
  }
  try {
    SC_CUDA(cudaSetDevice(c->device));
    if (c->world == 1) {
      gather_dofs(c, c->d_u[c->cur], c->d_out);
    } else {
      SC_CUDA(cudaMemsetAsync(c->d_out, 0, sizeof(double) * c->n_dof, c->stream));
      gather_owned(c, c->d_u[c->cur], c->d_out);
    }
    std::vector<double> tmp(c->n_dof);
    SC_CUDA(cudaMemcpyAsync(tmp.data(), c->d_out, sizeof(double) * c->n_dof, cudaMemcpyDeviceToHost, c->stream));
    const sc_status st = sc_sync(c);
    if (c->world == 1) {
      std::memcpy(u, tmp.data(), sizeof(double) * c->n_dof);
    } else {
      for (int32_t i : c->own_dofs) u[i] = tmp[i];
    }
    return st;
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_exchange_local(sc_ctx* const* ctxs, int32_t world) {
  if (!ctxs || world < 1) return SC_ERR_STATE;
  sc_ctx* c0 = ctxs[0];
  try {
    for (int r = 0; r < world; ++r) {
      if (!ctxs[r] || ctxs[r]->world != world || ctxs[r]->rank != r || ctxs[r]->nccl_comm)
        throw ScError(SC_ERR_CONFIG, "sc_exchange_local: ctxs[r] must be rank r of an in-process group");
      if (ctxs[r]->host_step != c0->host_step) throw ScError(SC_ERR_STATE, "ranks at different steps");
    }
    for (int r = 0; r < world; ++r) {
      SC_CUDA(cudaSetDevice(ctxs[r]->device));
      SC_CUDA(cudaStreamSynchronize(ctxs[r]->stream));
    }
    for (int q = 0; q < world; ++q) {
      sc_ctx* d = ctxs[q];
      SC_CUDA(cudaSetDevice(d->device));
      for (int r = 0; r < world; ++r) {
        if (r == q) continue;
        const sc_ctx* src = ctxs[r];
        const int64_t n = d->xr_off[r + 1] - d->xr_off[r];
        if (n != src->xs_off[q + 1] - src->xs_off[q]) throw ScError(SC_ERR_STATE, "exchange lists disagree");
        if (n)
          SC_CUDA(cudaMemcpyAsync(d->d_xr_buf + d->xr_off[r], src->d_xs_buf + src->xs_off[q], sizeof(double) * n,
                                  cudaMemcpyDefault, d->stream));
      }
      enqueue_unpack(d, d->d_u[d->cur], d->stream);
      SC_CUDA(cudaStreamSynchronize(d->stream));
    }
    return SC_OK;
  } catch (const ScError& e) {
    return fail(c0, e);
  }
}

extern "C" sc_status sc_elastic_energy(sc_ctx* c, double* energy) {
  if (!c || !energy) return SC_ERR_STATE;
  if (c->world > 1) {
    c->err = "sc_elastic_energy: one rank";
    return SC_ERR_CONFIG;
  }
  try {
    SC_CUDA(cudaSetDevice(c->device));
    *energy = elastic_energy(c);
    return SC_OK;
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_estimate_dt(sc_ctx* c, int32_t iters, double* lambda_max, double* dt_crit) {
  if (!c) return SC_ERR_STATE;
  if (iters < 1 || c->world > 1 || c->integrator == 2) {
    c->err = "sc_estimate_dt: iters >= 1, one rank, an explicit or IMEX integrator";
    return SC_ERR_CONFIG;
  }
  try {
    SC_CUDA(cudaSetDevice(c->device));
    const double lam = estimate_lambda(c, iters);
    if (lambda_max) *lambda_max = lam;
    if (dt_crit) *dt_crit = lam > 0.0 ? 2.0 / std::sqrt(lam) : 0.0;
    return SC_OK;
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_set_receivers(sc_ctx* c, const double* xyz, int32_t n, int64_t capacity) {
  if (!c) return SC_ERR_STATE;
  if (n < 0 || (n > 0 && (!xyz || capacity < 1)) || c->world > 1) {
    c->err = "sc_set_receivers: n >= 0 points (xyz[3n]), capacity >= 1 rows, one rank";
    return SC_ERR_CONFIG;
  }
  try {
    SC_CUDA(cudaSetDevice(c->device));
    SC_CUDA(cudaStreamSynchronize(c->stream));
    const int nb = c->nb;
    std::vector<int32_t> lat((size_t)n * nb, 0);
    std::vector<double> w((size_t)n * nb, 0.0);
    std::vector<std::pair<int64_t, double>> pw;
    for (int r = 0; r < n; ++r) {
      point_weights(c, xyz + 3 * (size_t)r, false, pw);
      for (size_t k = 0; k < pw.size(); ++k) {
        lat[(size_t)r * nb + k] = (int32_t)pw[k].first;
        w[(size_t)r * nb + k] = pw[k].second;
      }
    }
    for (void* p : {(void*)c->d_rec_lat, (void*)c->d_rec_w, (void*)c->d_rec_trace})
      if (p) cudaFree(p);
    c->d_rec_lat = nullptr;
    c->d_rec_w = nullptr;
    c->d_rec_trace = nullptr;
    c->n_rec = n;
    c->rec_cap = n ? capacity : 0;
    if (n) {
      SC_CUDA(cudaMalloc(&c->d_rec_lat, sizeof(int32_t) * lat.size()));
      SC_CUDA(cudaMalloc(&c->d_rec_w, sizeof(double) * w.size()));
      SC_CUDA(cudaMalloc(&c->d_rec_trace, sizeof(double) * (size_t)n * capacity));
      SC_CUDA(cudaMemcpy(c->d_rec_lat, lat.data(), sizeof(int32_t) * lat.size(), cudaMemcpyHostToDevice));
      SC_CUDA(cudaMemcpy(c->d_rec_w, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice));
      SC_CUDA(cudaMemset(c->d_rec_trace, 0, sizeof(double) * (size_t)n * capacity));
    }
    destroy_graphs(c);
    build_graphs(c);
    return SC_OK;
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_read_traces(sc_ctx* c, double* out, int64_t max_rows, int64_t* rows) {
  if (!c) return SC_ERR_STATE;
  try {
    SC_CUDA(cudaSetDevice(c->device));
    const int64_t nr = std::min<int64_t>(std::min<int64_t>(c->host_step, c->rec_cap), std::max<int64_t>(0, max_rows));
    if (rows) *rows = nr;
    if (nr > 0 && c->n_rec > 0 && out)
      SC_CUDA(cudaMemcpyAsync(out, c->d_rec_trace, sizeof(double) * nr * c->n_rec, cudaMemcpyDeviceToHost, c->stream));
    return sc_sync(c);
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_nccl_unique_id(void* out128) {
  try {
    nccl_unique_id(out128);
    return SC_OK;
  } catch (const ScError& e) {
    g_setup_err = e.msg;
    return e.st;
  }
}

extern "C" sc_status sc_read_c_state(sc_ctx* c, double* v_c, double* a_c, int64_t len) {
  if (!c) return SC_ERR_STATE;
  if (len < c->n_c) {
    c->err = "output buffer too small";
    return SC_ERR_CONFIG;
  }
  try {
    SC_CUDA(cudaSetDevice(c->device));
    std::vector<double> tmp(c->n_cl);
    for (int which = 0; which < 2; ++which) {
      double* dst = which == 0 ? v_c : a_c;
      if (!dst || c->n_cl == 0) continue;
      SC_CUDA(cudaMemcpyAsync(tmp.data(), which == 0 ? c->d_vc : c->d_ac, sizeof(double) * c->n_cl,
                              cudaMemcpyDeviceToHost, c->stream));
      SC_CUDA(cudaStreamSynchronize(c->stream));
      for (int64_t i = 0; i < c->n_cl; ++i) dst[c->c_canon[i]] = tmp[i];
    }
    return SC_OK;
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_cell_dt(sc_ctx* c, int32_t which, double* dt_cell, int64_t len) {
  if (!c) return SC_ERR_STATE;
  if (which != 0 && which != 1) {
    c->err = "sc_cell_dt: which must be 0 (consistent mass) or 1 (HRZ-lumped mass)";
    return SC_ERR_CONFIG;
  }
  if (!dt_cell || len < c->n_cells) {
    c->err = "sc_cell_dt: output buffer too small (need prod(cells))";
    return SC_ERR_CONFIG;
  }
  try {
    SC_CUDA(cudaSetDevice(c->device));
    std::vector<double> cut(2 * (size_t)c->n_cut);
    if (c->n_cut)
      SC_CUDA(cudaMemcpy(cut.data(), c->d_cut_dt, sizeof(double) * cut.size(), cudaMemcpyDeviceToHost));
    size_t k = 0;   // cut cells in ascending cell order (c->cut_cells)
    for (int64_t i = 0; i < c->n_cells; ++i) {
      const int8_t cl = c->cell_class[i];
      dt_cell[i] = cl == 0 ? c->dt_crit_uncut : (cl == 1 ? cut[2 * k++ + which] : 0.0);
    }
    return SC_OK;
  } catch (const ScError& e) {
    return fail(c, e);
  }
}

extern "C" sc_status sc_query(sc_ctx* c, sc_info* o) {
  if (!c || !o) return SC_ERR_STATE;
  std::memset(o, 0, sizeof(*o));
  o->n_dof = c->n_dof;
  o->n_d = c->n_d;
  o->n_c = c->n_c;
  o->n_irregular = c->n_irr;
  o->cells_uncut = c->cells_uncut;
  o->cells_cut = c->cells_cut;
  o->cells_empty = c->cells_empty;
  o->n_components = c->n_components;
  o->n_supernodes = c->n_sn;
  o->nnz_factor = c->nnz_factor;
  o->factor_height = c->height;
  o->dt = c->dt;
  o->dt_crit_uncut = c->dt_crit_uncut;
  o->step = c->host_step;
  o->bytes_per_step = c->bytes_per_step;
  o->bytes_explicit_per_step = c->bytes_explicit;
  o->kernels_per_step = c->kernels_per_step;
  o->lattice_nodes = c->n_lat;
  o->setup_seconds = c->setup_seconds;
  o->n_near = c->n_near;
  o->bytes_solve_per_step = c->bytes_solve;
  o->rank = c->rank;
  o->world = c->world;
  o->n_c_local = c->n_cl;
  o->halo_send = c->xs_off.empty() ? 0 : c->xs_off.back();
  o->halo_recv = c->xr_off.empty() ? 0 : c->xr_off.back();
  o->n_owned = c->world > 1 ? (int64_t)c->own_dofs.size() : c->n_dof;
  o->bytes_celem_per_step = c->bytes_celem;
  return SC_OK;
}

extern "C" sc_status sc_read_classification(sc_ctx* c, int8_t* cell_class, uint8_t* dof_is_c,
                                            int64_t* dof_lattice_index) {
  if (!c) return SC_ERR_STATE;
  if (cell_class) std::memcpy(cell_class, c->cell_class.data(), c->cell_class.size());
  for (int64_t i = 0; i < c->n_dof; ++i) {
    if (dof_is_c) dof_is_c[i] = c->ntype[c->dof_lat[i]] == 3 ? 1 : 0;
    if (dof_lattice_index) dof_lattice_index[i] = c->dof_lat[i];
  }
  return SC_OK;
}

extern "C" sc_status sc_dof_coords(sc_ctx* c, double* xyz, int64_t len) {
  if (!c) return SC_ERR_STATE;
  if (!xyz || len < 3 * c->n_dof) {
    c->err = "output buffer too small";
    return SC_ERR_CONFIG;
  }
  const GridP& g = c->g;
  for (int64_t i = 0; i < c->n_dof; ++i) {
    int64_t lat = c->dof_lat[i];
    for (int k = 0; k < 3; ++k) {
      double x = 0.0;
      if (k < g.dim) {
        int64_t j = lat % g.nl[k];
        lat /= g.nl[k];
        int64_t e = std::min<int64_t>(j / g.p, g.N[k] - 1);
        int64_t l = j - e * g.p;
        x = g.lo[k] + g.h[k] * (e + (c->gll_x[l] + 1.0) * 0.5);
      }
      xyz[3 * i + k] = x;
    }
  }
  return SC_OK;
}

extern "C" const char* sc_last_error(const sc_ctx* c) { return c ? c->err.c_str() : g_setup_err.c_str(); }

extern "C" void sc_destroy(sc_ctx* c) { free_ctx(c); }

extern "C" sc_status sc_profile(sc_ctx* c, int32_t which, int64_t n) {
  if (!c) return SC_ERR_STATE;
  if (which < 0 || which > 3 || n < 0) {
    c->err = "sc_profile: which in {0,1,2,3}, n >= 0";
    return SC_ERR_CONFIG;
  }
  try {
    SC_CUDA(cudaSetDevice(c->device));
    for (int64_t i = 0; i < n; ++i) profile_launch(c, which);
    return SC_OK;
  } catch (const ScError& e) {
    return fail(c, e);
  }
}
