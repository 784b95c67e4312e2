// Internal definitions of libsc (product path).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/sc.h"

#define SC_MAXP1 9            // p <= 8
#define SC_MAX_VOIDS 4096
// solve work items (solve.cu, factor.cpp): one staging buffer of SOLVE_STAGE doubles per CTA;
// forward tiles have at most SOLVE_TILE columns, backward tiles at most SOLVE_BROWS rows
#define SOLVE_TILE 128
#define SOLVE_STAGE 4096
#ifndef SOLVE_BROWS
#define SOLVE_BROWS 512
#endif
#ifndef SOLVE_NT
#define SOLVE_NT 192     // k_solve threads: 4 compute warps + claimer + publisher
#endif
#ifndef SOLVE_MINB
#define SOLVE_MINB 6     // resident k_solve CTAs per SM (shared memory: 32 KB stage + 4 KB)
#endif

// ---------------------------------------------------------------- device-side data
struct DVoid {
  int kind;
  double c[3];
  double A[6];
  double n[3];
  double b;
  double bblo[3], bbhi[3];  // inflated bounding box (ellipsoids): exact-safe culling
};

// geometry/lattice parameters passed by value to kernels
struct GridP {
  int dim, p, s, depth;
  int N[3];
  int64_t nl[3];       // lattice nodes per axis (N*p+1; 1 for unused axes)
  double lo[3], hi[3];
  double h[3];
  int ezl;             // 3D explicit tiles: element layers per tile along z (step.cu)
};

// device view of the supernodal factor structure + persistent-solve work list (solve.cu)
struct SolveDev {
  const int4* items;           // 5 x int4 per item (factor.cpp)
  int n_items, n_sn;
  const int32_t *w, *r, *c0, *goff, *gptr, *gidx, *uoff, *roff, *R;
  const int2* g2;              // front gather lists inline (<= 2 entries; factor.cpp)
  const int64_t* aoff;         // per supernode offset of its stacked [D_s; G_s] panel
  const int32_t *nblk;         // [2][n_sn] 32-blocks per phase (0 forward, 1 backward)
  const int32_t *chptr, *chidx, *parent;
  const double* A;             // stacked panels, ld x w column-major each (factor.cpp panel_ld)
  double *U, *b, *q, *x;
  double* part;                // tile partial sums
  int* cnt;                    // [2][n_sn] completed blocks per phase
  int* done_ch;                // [n_sn] children whose forward phase is complete
  int* bcnt;                   // per block: tiles done (ticket)
  int* ready;                  // ready queue slots: item + 1 (0 = not yet pushed)
  int* head;                   // ready-queue consumer counter
  int* tail;                   // ready-queue producer counter
  const int32_t *item_first, *item_cnt;   // [2][n_sn] item range of each phase
  const int32_t* nch;          // [n_sn] number of children
  const int32_t* init;         // forward items of the leaves (ready at launch)
  int n_init;
  int tile;                    // reduction-tile length (SOLVE_TILE)
  int stage;                   // staging buffer (doubles; two per CTA)
  unsigned long long* trace;   // optional (SC_TRACE): per item [claim, item, gathered, staged, done] ns
};

// Device factor of one SPD matrix (S or M^cc), shared symbolic structure.  For supernode s
// with L = [L_ss 0; L_Rs L_RR] the panel stores D_s = (L_ss L_ss^T)^{-1} (w x w, full) on
// top of G_s = L_Rs L_ss^{-1} (r x w): forward  q_s = D_s v_s, U_s = G_s v_s (+ children);
// backward x_s = q_s - G_s^T x_R  (solve.cu).
struct Factor {
  double* A = nullptr;     // stacked panels [D_s; 0; G_s; 0], column-major (factor.cpp make_panel)
  double* d = nullptr;     // Jacobi scaling: the factor is of D A D, D = diag(A)^{-1/2}
};

struct sc_ctx {
  std::string err;
  // ---- problem
  GridP g;
  int nb = 0;               // (p+1)^dim
  double alpha = 0, rho = 1, c = 1, dt = 0, fill_eps = 1e-10;
  int integrator = 0;       // 0 Newmark IMEX; 1 CDM with HRZ-lumped cut cells (NEXT-1(c)); 4 leap-frog
  int lf_m = 1;             // integrator 4: substeps of the cut DOFs per step
  int lf_coupling = 0;      // integrator 4: 0 interpolated d values, 1 frozen (reading LF3)
  double* d_mc = nullptr;   // integrator 1: HRZ-lumped mass of the c DOFs (ND order)
  std::vector<DVoid> voids;
  int64_t n_cells = 0, n_lat = 0;
  // rules (host, own implementation)
  std::vector<double> gll_x, gll_w, gau_x, gau_w, Mhat, Khat;   // Mhat/Khat (p+1)^2 row-major
  std::vector<double> Kref;                                     // nb x nb uncut K_e
  std::vector<double> Mref;                                     // nb uncut lumped diag
  double dt_crit_uncut = 0;
  // ---- classification (host copies)
  std::vector<int8_t> cell_class;     // 0 uncut 1 cut 2 empty
  std::vector<uint8_t> ntype;         // per lattice node: 0 hole 1 tensor-d far from c 2 irregular-d 3 c
                                      // 4 tensor-d sharing an element with a c node ("near")
  std::vector<int64_t> dof_lat;       // canonical DOFs -> lattice index
  int64_t n_dof = 0, n_d = 0, n_c = 0, n_irr = 0, n_near = 0;
  int64_t cells_uncut = 0, cells_cut = 0, cells_empty = 0;
  // c numbering: ND order (new index) -> lattice index; canonical c order map
  std::vector<int64_t> c_lat;         // ND order
  std::vector<int32_t> c_canon;       // ND index -> rank among c DOFs in canonical order
  // ---- device state
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  DVoid* d_voids = nullptr;
  double* d_u[2] = {nullptr, nullptr};     // lattice buffers (A,B)
  int cur = 0;                             // d_u[cur] holds u_n
  uint8_t* d_ntype = nullptr;
  int8_t* d_cell_class = nullptr;
  int64_t* d_dof_lat = nullptr;
  double* d_out = nullptr;                 // n_dof gather buffer for sc_read (and u0 staging)
  double* d_stage = nullptr;               // n_dof staging buffer of v0 (allocated on first use)
  double* d_vlat = nullptr;                // lattice v0 of the start (allocated on first use)
  double* d_ft = nullptr;                  // f_t series
  int64_t n_t = 0;
  long long* d_step = nullptr;             // device step counter
  int* d_flag = nullptr;                   // non-finite flag
  int64_t host_step = 0;
  // irregular d nodes
  int32_t* d_irr_lat = nullptr;
  double* d_irr_invm = nullptr;
  double* d_irr_fx = nullptr;
  // tensor-d nodes carrying a distributed load (source kind 2): lattice index, f_x / M_ii
  int32_t* d_load_lat = nullptr;
  double* d_load_fxm = nullptr;
  int64_t n_load = 0;
  double* d_Kref = nullptr;
  // c state (ND order)
  int32_t* d_c_lat = nullptr;
  double *d_vc = nullptr, *d_ac = nullptr, *d_fxc = nullptr;
  double *d_b = nullptr, *d_q = nullptr, *d_x = nullptr, *d_U = nullptr;
  // c elements
  int64_t n_celem = 0, n_cut = 0;
  int32_t* d_celem_cell = nullptr;   // cell index of each c-element
  int32_t* d_celem_kidx = nullptr;   // index into d_Kcut or -1 (uncut -> Kref)
  int32_t* d_celem_cidx = nullptr;   // [e*nb + loc] c index (ND) or -1
  int64_t n_celem_cut = 0, n_celem_ref = 0;
  int32_t* d_celem_cut_ids = nullptr;   // c elements with a dense cut K_e
  int32_t* d_celem_ref_ids = nullptr;   // uncut c elements (reference K_e)
  double* d_Kcut = nullptr;          // n_cut x nb x nb (setup; dropped once packed)
  double* d_Kpk = nullptr;           // n_cut x nb(nb+1)/2: packed lower triangles (step)
  double* d_cut_dt = nullptr;        // [n_cut][2] cell-wise critical step (consistent, HRZ) of the cut cells
  int ct_T = 0, ct_nt = 0, ct_TS = 0;   // tiles: T rows, nt per dimension, TS doubles (stride)
  long long ct_ms = 0;                  // doubles per stored matrix
  double* d_Y = nullptr;             // n_celem x nb
  int32_t *d_rhs_ptr = nullptr, *d_rhs_idx = nullptr;   // c node -> Y entries
  // factor structure (shared by S and M^cc)
  int n_sn = 0, height = 0;
  int32_t *d_sn_c0 = nullptr, *d_sn_w = nullptr, *d_sn_r = nullptr;
  int64_t* d_sn_aoff = nullptr;
  int32_t *d_sn_roff = nullptr, *d_sn_uoff = nullptr, *d_sn_goff = nullptr;
  int32_t* d_R = nullptr;             // row structures (ND c indices)
  int32_t *d_gptr = nullptr, *d_gidx = nullptr, *d_g2 = nullptr;
  int32_t* d_items = nullptr;         // int4 work items
  int32_t *d_nitem = nullptr, *d_chptr = nullptr, *d_chidx = nullptr, *d_parent = nullptr;
  int32_t* d_qmeta = nullptr;         // ready-queue metadata (solve.cu)
  int n_init = 0;
  int* d_solve_cnt = nullptr;         // [2*n_sn] phase counters, [n_bctr] tickets, head
  double* d_part = nullptr;           // tile partials
  int n_items = 0, solve_grid = 0, solve_stage = SOLVE_STAGE;
  unsigned long long* d_trace = nullptr;   // SC_TRACE: solve item timeline (debug)
  std::vector<int32_t> h_items;            // host copy of the work list (debug)
  size_t n_counters = 0;
  SolveDev solve_dev{};
  Factor fS, fM;
  int64_t nnz_factor = 0;   // sum_s w_s (w_s + r_s): stored panel entries
  int64_t nnz_G = 0;        // sum_s r_s w_s (re-read by the backward sweep)
  int64_t sum_r = 0;        // sum_s r_s (update-vector entries)
  int64_t n_components = 0;
  // near-d tiles of the explicit kernel (tile ids, x fastest)
  uint8_t* d_clean = nullptr;         // 3D: per explicit tile, 1 = owns only tensor-d nodes
  int* d_near_tiles = nullptr;
  int n_near_tiles = 0;
  // graphs and the step pipeline (step.cu)
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  cudaStream_t s_hi = nullptr;             // high-priority stream of the c part
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t s_ref = nullptr;            // side stream of the reference-element products
  cudaEvent_t ev_ref0 = nullptr, ev_ref1 = nullptr;
  bool far_ready = false;                  // far-d update of the current step already enqueued
  bool pipelined = false;                  // SC_PIPELINE: far-d update forked against the c part
  int far_cap = 0;                         // resident CTAs per SM of the forked far-d update (0 = no cap)
  int solve_cap = 0;                       // resident solve CTAs per SM (0 = occupancy limit)
  int kernels_per_step = 0;
  double bytes_per_step = 0, bytes_explicit = 0, bytes_solve = 0, bytes_celem = 0;
  double setup_seconds = 0;
  // setup scratch
  int src_kind = 0;
  double src_x[3] = {0, 0, 0};
  std::vector<double> Kcut_host, Mcut_host;   // freed after the factorisation
  std::vector<long long> cut_cells;           // ascending cell index of each cut cell
  std::vector<std::vector<unsigned long long>> cut_leaves;   // source kind 2: spacetree leaves per cut cell
  double src_sigma = 0.0, src_amp = 0.0;      // source kind 2: Gaussian bell width, amplitude
  int max_w = 0;                              // widest supernode
  double* d_tmp = nullptr;
  // ---- multi-rank slab decomposition (partition.cpp; world > 1)
  int rank = 0, world = 1;
  std::vector<int> layer_lo;          // [world + 1] slab boundaries (element layers, split axis)
  std::vector<int> reg_lo, reg_hi;    // [world] compute regions (element layers)
  int64_t n_cl = 0;                   // c DOFs of this rank's components (device c part)
  std::vector<uint8_t> ntype_rank;    // node types this rank updates (0 elsewhere)
  int* d_far_tiles = nullptr;         // world > 1: explicit tiles holding this rank's far-d nodes
  int n_far_tiles = 0;
  // exchange after each step: per peer q, send (owned, needed by q) / receive lattice indices
  std::vector<int64_t> xs_off, xr_off;   // [world + 1]
  int32_t *d_xs_idx = nullptr, *d_xr_idx = nullptr;
  double *d_xs_buf = nullptr, *d_xr_buf = nullptr;
  std::vector<int32_t> own_dofs;      // canonical DOF indices owned by this rank
  int32_t* d_own_lat = nullptr;       // their lattice indices
  int32_t* d_own_dof = nullptr;
  void* nccl_comm = nullptr;          // ncclComm_t (world > 1 with an NCCL unique id)
  double* d_full = nullptr;           // n_dof reduction buffer of sc_read (NCCL)
  // receivers (NEXT-3): u(x_r, t_{n+1}) = sum_i N_i(x_r) u_i recorded after every step
  int n_rec = 0;
  int64_t rec_cap = 0;
  int32_t* d_rec_lat = nullptr;       // [n_rec][nb] lattice indices (0 for padding)
  double* d_rec_w = nullptr;          // [n_rec][nb] basis values (0 for padding)
  double* d_rec_trace = nullptr;      // [rec_cap][n_rec]
};

// component summary for the partition plan (element layers of the split axis)
struct CompSpan {
  int lmin, lmax, centroid;
  double cost;
};

// ---------------------------------------------------------------- helpers
// Experiment knobs (schedule / ordering / variant switches): read from the environment ONLY in
// experiment builds (SC_NVCC_DEFS=-DSC_EXPERIMENTS with an SC_BUILD_TAG / SC_BUILD_OUT).  The
// product library ignores the environment except the SC_TRACE / SC_DEBUG diagnostics, which
// change no result.
inline const char* sc_knob(const char* name) {
#ifdef SC_EXPERIMENTS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

#define SC_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e__ = (call);                                                          \
    if (e__ != cudaSuccess) {                                                          \
      throw ScError(SC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
    }                                                                                  \
  } while (0)

struct ScError {
  sc_status st;
  std::string msg;
  ScError(sc_status s, std::string m) : st(s), msg(std::move(m)) {}
};

// host rules (rules.cpp)
void host_gll(int p, std::vector<double>& x, std::vector<double>& w);
void host_gauss(int n, std::vector<double>& x, std::vector<double>& w);
void host_lagrange(const std::vector<double>& nodes, double xi, double* v, double* dv);
void host_reference(sc_ctx* c);
bool host_phys(const std::vector<DVoid>& voids, const double x[3]);
double host_lattice(double lo, double hi, int64_t m, int64_t den);

// setup (setup.cu)
void setup_device_geometry(sc_ctx* c);
// partition (partition.cpp)
void plan_partition(sc_ctx* c, const std::vector<CompSpan>& comps, std::vector<int>& owner);
bool region_computes_plane(const sc_ctx* c, int q, int64_t z);
int plane_owner(const sc_ctx* c, int64_t z);
void build_exchange(sc_ctx* c, const std::vector<int>& c_owner_of_lat_sorted_idx,
                    const std::vector<int64_t>& clat_global);
// NCCL transport (nccl.cpp; dlopen'ed, world > 1 with a unique id)
void nccl_init(sc_ctx* c, const void* unique_id);
void nccl_exchange(sc_ctx* c);
void nccl_allreduce_sum(sc_ctx* c, double* buf, int64_t n);
void nccl_destroy(sc_ctx* c);
int nccl_unique_id(void* out128);
// exchange kernels (step.cu)
void enqueue_pack(sc_ctx* c, const double* u, cudaStream_t st);
void enqueue_unpack(sc_ctx* c, double* u, cudaStream_t st);
void gather_owned(sc_ctx* c, const double* d_lat, double* d_dst);
double estimate_lambda(sc_ctx* c, int iters);
double elastic_energy(sc_ctx* c);
// factor (factor.cpp)
void setup_factor(sc_ctx* c, const std::vector<double>& Mcut_host);
void point_weights(const sc_ctx* c, const double* x, bool with_alpha,
                   std::vector<std::pair<int64_t, double>>& out);
void bell_weights(const sc_ctx* c, std::vector<std::pair<int64_t, double>>& out);
// step (step.cu)
void setup_step_structures(sc_ctx* c);
void explicit_tiling(const GridP& g, int ext[3], int tg[3]);
void explicit_prepare(sc_ctx* c);
void build_graphs(sc_ctx* c);
void destroy_graphs(sc_ctx* c);
void run_startup(sc_ctx* c, const double* u0, const double* v0);
void enqueue_step(sc_ctx* c, int parity, cudaStream_t st);
void enqueue_far_prologue(sc_ctx* c);
void launch_solve(sc_ctx* c, const Factor& f, cudaStream_t st);
void device_upload_reference(sc_ctx* c);
void gather_dofs(sc_ctx* c, const double* d_lat, double* d_out);

void profile_launch(sc_ctx* c, int which);
