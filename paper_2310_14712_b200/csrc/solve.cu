// (a5) implicit cut-DOF solve S a^c_{n+1} = r^c with the factor computed once at setup
// ("triangular matrix system with the factorized system
// matrix S" each step).  The factor is of the Jacobi-scaled matrix D S D (factor.cpp).
//
// One persistent kernel performs both sweeps.  Every supernode GEMV is cut into tiles
// (forward: 32 rows x 256 columns, backward: 32 outputs x 256 rows); a tile writes its 32
// partial sums to a private slot, and the LAST tile of each 32-wide block (atomic ticket)
// sums the block's partials in fixed tile order -> deterministic results.  Tiles are stored
// in a topological order (forward by supernode height, backward by height descending);
// CTAs dequeue them from a global counter and spin until the phase counters they depend
// on are complete.  Every dependency points to an EARLIER tile and tiles are only dequeued
// by running CTAs, so all producers are resident: no deadlock, no cooperative launch.
// Producer: partials / results, __threadfence, atomicAdd.  Consumer: spin, __threadfence,
// reads of produced data with ld.global.cg (L1 bypass).
//
// Phases per supernode s (w columns, r rows below, c0 first column):
//  fA: y_s = L_ss^{-1} (b_s - child updates)            tiles over (row block, column tile)
//  fB: U_s = child updates + L_{R,s} y_s                  tiles over (row block, column tile)
//  bA: z_s = y_s - L_{R,s}^T x[R_s]                       tiles over (column block, row tile)
//  bB: x_s = L_ss^{-T} z_s                                tiles over (output block, row tile)
#include "sc_internal.h"

namespace {

enum { IT_FA = 0, IT_FB = 1, IT_BA = 2, IT_BB = 3, IT_FF = 4, IT_BF = 5 };
constexpr int TILE = 256;  // columns (forward) / rows (backward) per tile

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// poll with plain acquire loads (no RMW traffic on the L2 atomic units) and backoff
__device__ __forceinline__ void wait_ge(const int* p, int target) {
  if (target <= 0) return;
  unsigned ns = 32;
  while (ld_acquire(p) < target) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

// sum_{j in [j0, j1) step js} A[i + j ld] v[j] for one row per lane, 8 loads in flight
__device__ __forceinline__ double row_dot(const double* A, size_t ld, int i, bool ok, int j0, int j1, int js,
                                          const double* v) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (ok) {
    int j = j0;
    for (; j + 7 * js < j1; j += 8 * js) {
      double x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = A[i + (size_t)(j + k * js) * ld];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k & 3] += x[k] * v[j + k * js];
    }
    for (; j < j1; j += js) acc[0] += A[i + (size_t)j * ld] * v[j];
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// sum_{q in [q0, q1) step 32} Ac[q] v[q] by one lane (column dot product, 8 loads in flight)
__device__ __forceinline__ double col_dot(const double* Ac, int q0, int q1, const double* v) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int q = q0;
  for (; q + 7 * 32 < q1; q += 256) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = Ac[q + 32 * k];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k & 3] += x[k] * v[q + 32 * k];
  }
  for (; q < q1; q += 32) acc[0] += Ac[q] * v[q];
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// y[0..nr) = A[0..nr, 0..nc) v  (A column-major, leading dimension ld; v, y in smem):
// each warp owns whole 32-row blocks (no cross-warp reduction, no barrier inside).
__device__ __forceinline__ void cta_gemv_rows(const double* A, int ld, int nr, int nc, const double* v, double* y,
                                              double (*)[33]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int rb = warp * 32; rb < nr; rb += 256) {
    const int i = rb + lane;
    const double t = row_dot(A, ld, i, i < nr, 0, nc, 1, v);
    if (i < nr) y[i] = t;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_solve(SolveDev a) {
  __shared__ double vs[TILE];
  __shared__ double part[8][33];
  __shared__ double fv[FUSE_W], fy[FUSE_W], fu[FUSE_R];   // fused small-supernode phases
  __shared__ int s_item, s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  while (true) {
    if (tid == 0) s_item = atomicAdd(a.head, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= a.n_items) return;
    const int4 d0 = a.items[2 * it], d1 = a.items[2 * it + 1];
    const int type = d0.x, s = d0.y, blk = d0.z, t = d0.w;   // blk: 32-block, t: tile in block
    const int ntb = d1.x, pslot = d1.y, bctr = d1.z, lo = d1.w;  // lo: first column/row of tile
    const int w = a.w[s], r = a.r[s], c0 = a.c0[s];
    const int n_sn = a.n_sn;
    // ---- dependencies
    if (tid == 0) {
      if (type == IT_FA || type == IT_FF) {
        for (int q = a.chptr[s]; q < a.chptr[s + 1]; ++q) {
          const int c = a.chidx[q];
          wait_ge(a.cnt + 1 * n_sn + c, a.nblk[1 * n_sn + c]);
        }
      } else if (type == IT_FB) {
        wait_ge(a.cnt + 0 * n_sn + s, a.nblk[0 * n_sn + s]);
      } else if (type == IT_BA || type == IT_BF) {
        const int p = a.parent[s];
        if (p >= 0) wait_ge(a.cnt + 3 * n_sn + p, a.nblk[3 * n_sn + p]);
        wait_ge(a.cnt + 0 * n_sn + s, a.nblk[0 * n_sn + s]);
      } else {
        wait_ge(a.cnt + 2 * n_sn + s, a.nblk[2 * n_sn + s]);
      }
      __threadfence();
    }
    __syncthreads();
    if (type == IT_FF) {
      // ---- fused forward phase of a small supernode (one CTA)
      const int go = a.goff[s];
      for (int j = tid; j < w; j += 256) {
        double v = a.b[c0 + j];
        for (int q = a.gptr[go + j]; q < a.gptr[go + j + 1]; ++q) v -= __ldcg(a.U + a.gidx[q]);
        fv[j] = v;
      }
      __syncthreads();
      cta_gemv_rows(a.Linv + a.linv_off[s], w, w, w, fv, fy, part);
      for (int j = tid; j < w; j += 256) a.y[c0 + j] = fy[j];
      if (r > 0) {
        cta_gemv_rows(a.LR + a.lr_off[s], r, r, w, fy, fu, part);
        for (int i = tid; i < r; i += 256) {
          double v = fu[i];
          for (int q = a.gptr[go + w + i]; q < a.gptr[go + w + i + 1]; ++q) v += __ldcg(a.U + a.gidx[q]);
          a.U[a.uoff[s] + i] = v;
        }
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        atomicAdd(a.cnt + 0 * n_sn + s, 1);
        atomicAdd(a.cnt + 1 * n_sn + s, 1);
      }
      continue;
    }
    if (type == IT_BF) {
      // ---- fused backward phase of a small supernode (one CTA)
      for (int i = tid; i < r; i += 256) fu[i] = __ldcg(a.x + a.R[a.roff[s] + i]);
      __syncthreads();
      const double* LR = a.LR + a.lr_off[s];
      for (int j = warp; j < w; j += 8) {
        double v = col_dot(LR + (size_t)j * r, lane, r, fu);
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) fv[j] = __ldcg(a.y + c0 + j) - v;
      }
      __syncthreads();
      const double* Li = a.Linv + a.linv_off[s];
      for (int i = warp; i < w; i += 8) {
        double v = 0.0;
        v = col_dot(Li + (size_t)i * w, i + lane, w, fv);
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) a.x[c0 + i] = v;
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        atomicAdd(a.cnt + 2 * n_sn + s, 1);
        atomicAdd(a.cnt + 3 * n_sn + s, 1);
      }
      continue;
    }
    double* P = a.part + pslot;   // this block's partials: [ntb][32]
    if (type == IT_FA || type == IT_FB) {
      // ---- row-oriented tile: rows blk*32 + lane, columns [lo, hi)
      const int nrows = (type == IT_FA) ? w : r;
      const int hi = (type == IT_FA) ? min(min(w, blk * 32 + 32), lo + TILE) : min(w, lo + TILE);
      const int ncols = hi - lo;
      const int go = a.goff[s];
      for (int j = tid; j < ncols; j += 256) {
        double v;
        if (type == IT_FA) {
          v = a.b[c0 + lo + j];
          for (int q = a.gptr[go + lo + j]; q < a.gptr[go + lo + j + 1]; ++q) v -= __ldcg(a.U + a.gidx[q]);
        } else {
          v = __ldcg(a.y + c0 + lo + j);
        }
        vs[j] = v;
      }
      __syncthreads();
      const int i = blk * 32 + lane;
      const int ld = nrows;
      const double* A = (type == IT_FA ? a.Linv + a.linv_off[s] : a.LR + a.lr_off[s]) + (size_t)lo * ld;
      // warp covers columns warp*32 .. warp*32+31 of the tile
      const int j0 = warp * 32, j1 = min(ncols, j0 + 32);
      part[warp][lane] = row_dot(A, ld, i, i < nrows, j0, j1, 1, vs);
      __syncthreads();
      if (warp == 0) {
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) v += part[k][lane];
        P[t * 32 + lane] = v;
      }
    } else {
      // ---- column-oriented tile: outputs (columns) blk*32 + o, rows [lo, hi)
      const int o0 = blk * 32;
      const int hi = (type == IT_BA) ? min(r, lo + TILE) : min(w, lo + TILE);
      const int nr = hi - lo;
      for (int j = tid; j < nr; j += 256)
        vs[j] = (type == IT_BA) ? __ldcg(a.x + a.R[a.roff[s] + lo + j]) : __ldcg(a.z + c0 + lo + j);
      __syncthreads();
      const int ld = (type == IT_BA) ? r : w;
      const double* A = (type == IT_BA ? a.LR + a.lr_off[s] : a.Linv + a.linv_off[s]);
      // warp handles 4 output columns; lanes stride rows
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int col = o0 + warp * 4 + cc;
        double v = 0.0;
        if (col < w) {
          const double* Ac = A + (size_t)col * ld + lo;
          v = col_dot(Ac, lane, nr, vs);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) P[t * 32 + warp * 4 + cc] = v;
      }
    }
    // ---- last tile of the block reduces the partials in tile order
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(a.bcnt + bctr, 1) == ntb - 1);
    __syncthreads();
    if (s_last) {
      __threadfence();
      if (tid < 32) {
        const int o = blk * 32 + tid;
        double v = 0.0;
        for (int k = 0; k < ntb; ++k) v += __ldcg(P + k * 32 + tid);
        if (type == IT_FA) {
          if (o < w) a.y[c0 + o] = v;
        } else if (type == IT_FB) {
          if (o < r) {
            const int go = a.goff[s];
            for (int q = a.gptr[go + w + o]; q < a.gptr[go + w + o + 1]; ++q) v += __ldcg(a.U + a.gidx[q]);
            a.U[a.uoff[s] + o] = v;
          }
        } else if (type == IT_BA) {
          if (o < w) a.z[c0 + o] = __ldcg(a.y + c0 + o) - v;
        } else {
          if (o < w) a.x[c0 + o] = v;
        }
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) atomicAdd(a.cnt + type * n_sn + s, 1);
    }
    __syncthreads();
  }
}

}  // namespace

void launch_solve(sc_ctx* c, const Factor& f) {
  if (c->n_c == 0 || c->n_items == 0) return;
  SolveDev a = c->solve_dev;
  a.Linv = f.Linv;
  a.LR = f.LR;
  SC_CUDA(cudaMemsetAsync(c->d_solve_cnt, 0, sizeof(int) * c->n_counters, c->stream));
  if (c->solve_grid == 0) {
    int per_sm = 0, sms = 0, dev = 0;
    SC_CUDA(cudaGetDevice(&dev));
    SC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve, 256, 0));
    c->solve_grid = std::max(1, std::min(c->n_items, per_sm * sms));
  }
  k_solve<<<c->solve_grid, 256, 0, c->stream>>>(a);
  SC_CUDA(cudaGetLastError());
}
