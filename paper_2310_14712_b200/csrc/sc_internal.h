// Internal definitions of libsc (product path).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sc.h"

#define SC_MAXP1 9            // p <= 8
#define SC_MAX_VOIDS 4096
// supernodes with w <= FUSE_W, r <= FUSE_R and (w*w + r*w) <= FUSE_ENTRIES are solved by a
// single CTA per sweep (solve.cu); larger ones are tiled
#define FUSE_W 128
#define FUSE_R 1024
#define FUSE_ENTRIES 16384

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
};

// device view of the supernodal factor structure + persistent-solve work list (solve.cu)
struct SolveDev {
  const int4* items;           // 2 x int4 per tile: (type, s, block, tile) (ntiles, pslot, bctr, lo)
  int n_items, n_sn;
  const int32_t *w, *r, *c0, *goff, *gptr, *gidx, *uoff, *roff, *R;
  const int64_t *linv_off, *lr_off;
  const int32_t *nblk;         // [4][n_sn] 32-blocks per phase
  const int32_t *chptr, *chidx, *parent;
  const double *Linv, *LR;
  double *U, *b, *y, *x, *z;
  double* part;                // tile partial sums
  int* cnt;                    // [4][n_sn] completed blocks per phase
  int* bcnt;                   // per block: tiles done (ticket)
  int* head;                   // dequeue counter
};

struct Factor {          // device factor of one SPD matrix (S or M^cc), shared symbolic
  double* Linv = nullptr;  // per supernode w x w column-major inverse of L_ss (lower)
  double* LR = nullptr;    // per supernode r x w column-major L_{R_s, s}
  double* d = nullptr;     // Jacobi scaling: the factor is of D A D, D = diag(A)^{-1/2}
};

struct sc_ctx {
  std::string err;
  // ---- problem
  GridP g;
  int nb = 0;               // (p+1)^dim
  double alpha = 0, rho = 1, c = 1, dt = 0, fill_eps = 1e-10;
  std::vector<DVoid> voids;
  int64_t n_cells = 0, n_lat = 0;
  // rules (host, own implementation)
  std::vector<double> gll_x, gll_w, gau_x, gau_w, Mhat, Khat;   // Mhat/Khat (p+1)^2 row-major
  std::vector<double> Kref;                                     // nb x nb uncut K_e
  std::vector<double> Mref;                                     // nb uncut lumped diag
  double dt_crit_uncut = 0;
  // ---- classification (host copies)
  std::vector<int8_t> cell_class;     // 0 uncut 1 cut 2 empty
  std::vector<uint8_t> ntype;         // per lattice node: 0 hole 1 tensor-d 2 irregular-d 3 c
  std::vector<int64_t> dof_lat;       // canonical DOFs -> lattice index
  int64_t n_dof = 0, n_d = 0, n_c = 0, n_irr = 0;
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
  double* d_out = nullptr;                 // n_dof gather buffer for sc_read
  double* d_ft = nullptr;                  // f_t series
  int64_t n_t = 0;
  long long* d_step = nullptr;             // device step counter
  int* d_flag = nullptr;                   // non-finite flag
  int64_t host_step = 0;
  // irregular d nodes
  int32_t* d_irr_lat = nullptr;
  double* d_irr_invm = nullptr;
  double* d_irr_fx = nullptr;
  double* d_Kref = nullptr;
  // c state (ND order)
  int32_t* d_c_lat = nullptr;
  double *d_vc = nullptr, *d_ac = nullptr, *d_fxc = nullptr;
  double *d_b = nullptr, *d_y = nullptr, *d_x = nullptr, *d_z = nullptr, *d_U = nullptr;
  // c elements
  int64_t n_celem = 0, n_cut = 0;
  int32_t* d_celem_cell = nullptr;   // cell index of each c-element
  int32_t* d_celem_kidx = nullptr;   // index into d_Kcut or -1 (uncut -> Kref)
  int32_t* d_celem_cidx = nullptr;   // [e*nb + loc] c index (ND) or -1
  double* d_Kcut = nullptr;          // n_cut x nb x nb
  double* d_Y = nullptr;             // n_celem x nb
  int32_t *d_rhs_ptr = nullptr, *d_rhs_idx = nullptr;   // c node -> Y entries
  // factor structure (shared by S and M^cc)
  int n_sn = 0, height = 0;
  int32_t *d_sn_c0 = nullptr, *d_sn_w = nullptr, *d_sn_r = nullptr;
  int64_t *d_sn_linv = nullptr, *d_sn_lr = nullptr;
  int32_t *d_sn_roff = nullptr, *d_sn_uoff = nullptr, *d_sn_goff = nullptr;
  int32_t* d_R = nullptr;             // row structures (ND c indices)
  int32_t *d_gptr = nullptr, *d_gidx = nullptr;
  int32_t* d_items = nullptr;         // int4 work items
  int32_t *d_nitem = nullptr, *d_chptr = nullptr, *d_chidx = nullptr, *d_parent = nullptr;
  int* d_solve_cnt = nullptr;         // [4*n_sn] phase counters, [n_bctr] tickets, head
  double* d_part = nullptr;           // tile partials
  int n_items = 0, solve_grid = 0;
  size_t n_counters = 0;
  SolveDev solve_dev{};
  Factor fS, fM;
  int64_t nnz_factor = 0;
  int64_t n_components = 0;
  // graphs
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  int kernels_per_step = 0;
  double bytes_per_step = 0, bytes_explicit = 0;
  double setup_seconds = 0;
  // setup scratch
  int src_kind = 0;
  double src_x[3] = {0, 0, 0};
  std::vector<double> Kcut_host, Mcut_host;   // freed after the factorisation
  std::vector<long long> cut_cells;           // ascending cell index of each cut cell
  int max_w = 0;                              // widest supernode
  double* d_tmp = nullptr;
  // multi-GPU (reserved)
  int rank = 0, world = 1;
};

// ---------------------------------------------------------------- helpers
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
// factor (factor.cpp)
void setup_factor(sc_ctx* c, const std::vector<double>& Mcut_host);
// step (step.cu)
void setup_step_structures(sc_ctx* c);
void build_graphs(sc_ctx* c);
void run_startup(sc_ctx* c, const double* u0, const double* v0);
void enqueue_step(sc_ctx* c, int parity);
void launch_solve(sc_ctx* c, const Factor& f);
void device_upload_reference(sc_ctx* c);
void gather_dofs(sc_ctx* c, const double* d_lat, double* d_out);
void profile_launch(sc_ctx* c, int which);
