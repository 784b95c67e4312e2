// (a5) implicit cut-DOF solve S a^c_{n+1} = r^c with the factor computed once at setup
// ("triangular matrix system with the factorized system
// matrix S" each step).
//
// One persistent kernel performs both sweeps.  Work items (supernode s, row/column chunk)
// are stored in a topological order (forward: by supernode height, phase A before B;
// backward: by height descending, phase A before B).  CTAs dequeue items from a global
// counter; an item spins until the counters of the items it depends on are complete.
// Every dependency points to an EARLIER item, and an item is only dequeued by a running
// CTA, so all producers are resident: no deadlock without a cooperative launch.
// Producer: writes results, __threadfence, atomicAdd(counter).  Consumer: spins on the
// counter, __threadfence, reads produced data with ld.global.cg (bypassing L1).
//
// Forward (multifrontal, deterministic):  fA: y_s = L_ss^{-1} (b_s - sum child updates)
//                                         fB: U_s = sum child updates + L_{R_s,s} y_s
// Backward:                               bA: z_s = y_s - L_{R_s,s}^T x[R_s]
//                                         bB: x_s = L_ss^{-T} z_s
#include "sc_internal.h"

namespace {

enum { IT_FA = 0, IT_FB = 1, IT_BA = 2, IT_BB = 3 };

__device__ __forceinline__ void wait_ge(const int* p, int target) {
  if (target <= 0) return;
  while (atomicAdd((int*)p, 0) < target) __nanosleep(32);
}

__global__ void __launch_bounds__(256) k_solve(SolveDev a) {
  extern __shared__ double sh[];  // [max_w]
  __shared__ double part[8][33];
  __shared__ int s_item;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    if (threadIdx.x == 0) s_item = atomicAdd(a.head, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= a.n_items) return;
    const int4 d = a.items[it];
    const int type = d.x, s = d.y, st = d.z;
    const int w = a.w[s], r = a.r[s], c0 = a.c0[s];
    // ---- wait for dependencies
    if (threadIdx.x == 0) {
      if (type == IT_FA) {
        for (int q = a.chptr[s]; q < a.chptr[s + 1]; ++q) {
          const int c = a.chidx[q];
          wait_ge(a.cnt + 1 * a.n_sn + c, a.nitem[1 * a.n_sn + c]);
        }
      } else if (type == IT_FB) {
        wait_ge(a.cnt + 0 * a.n_sn + s, a.nitem[0 * a.n_sn + s]);
      } else if (type == IT_BA) {
        const int p = a.parent[s];
        if (p >= 0) wait_ge(a.cnt + 3 * a.n_sn + p, a.nitem[3 * a.n_sn + p]);
        // y_s of the forward sweep is complete once all fB items were dequeued and done:
        wait_ge(a.cnt + 1 * a.n_sn + s, a.nitem[1 * a.n_sn + s]);
        wait_ge(a.cnt + 0 * a.n_sn + s, a.nitem[0 * a.n_sn + s]);
      } else {
        wait_ge(a.cnt + 2 * a.n_sn + s, a.nitem[2 * a.n_sn + s]);
      }
      __threadfence();
    }
    __syncthreads();
    if (type == IT_FA) {
      const int go = a.goff[s];
      for (int t = threadIdx.x; t < w; t += blockDim.x) {
        double f = a.b[c0 + t];
        for (int q = a.gptr[go + t]; q < a.gptr[go + t + 1]; ++q) f -= __ldcg(a.U + a.gidx[q]);
        sh[t] = f;
      }
      __syncthreads();
      const int i = st + lane;
      const int jmax = min(w, st + 32);
      const double* L = a.Linv + a.linv_off[s];
      double acc0 = 0.0, acc1 = 0.0;
      if (i < w) {
        int j = warp;
        for (; j + 8 < jmax; j += 16) {
          acc0 += L[i + (size_t)j * w] * sh[j];
          acc1 += L[i + (size_t)(j + 8) * w] * sh[j + 8];
        }
        if (j < jmax) acc0 += L[i + (size_t)j * w] * sh[j];
      }
      part[warp][lane] = acc0 + acc1;
      __syncthreads();
      if (warp == 0 && i < w) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += part[k][lane];
        a.y[c0 + i] = t;
      }
    } else if (type == IT_FB) {
      for (int t = threadIdx.x; t < w; t += blockDim.x) sh[t] = __ldcg(a.y + c0 + t);
      __syncthreads();
      const int i = st + lane;
      const double* L = a.LR + a.lr_off[s];
      double acc0 = 0.0, acc1 = 0.0;
      if (i < r) {
        int j = warp;
        for (; j + 8 < w; j += 16) {
          acc0 += L[i + (size_t)j * r] * sh[j];
          acc1 += L[i + (size_t)(j + 8) * r] * sh[j + 8];
        }
        if (j < w) acc0 += L[i + (size_t)j * r] * sh[j];
      }
      part[warp][lane] = acc0 + acc1;
      __syncthreads();
      if (warp == 0 && i < r) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += part[k][lane];
        const int go = a.goff[s];
        for (int q = a.gptr[go + w + i]; q < a.gptr[go + w + i + 1]; ++q) t += __ldcg(a.U + a.gidx[q]);
        a.U[a.uoff[s] + i] = t;
      }
    } else if (type == IT_BA) {
      const int j = st + warp;
      if (j < w) {
        const double* L = a.LR + a.lr_off[s] + (size_t)j * r;
        const int32_t* R = a.R + a.roff[s];
        double acc = 0.0;
        for (int i = lane; i < r; i += 32) acc += L[i] * __ldcg(a.x + R[i]);
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) a.z[c0 + j] = __ldcg(a.y + c0 + j) - acc;
      }
    } else {
      const int i = st + warp;
      if (i < w) {
        const double* L = a.Linv + a.linv_off[s] + (size_t)i * w;
        double acc = 0.0;
        for (int j = i + lane; j < w; j += 32) acc += L[j] * __ldcg(a.z + c0 + j);
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) a.x[c0 + i] = acc;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(a.cnt + type * a.n_sn + s, 1);
    }
  }
}

}  // namespace

void launch_solve(sc_ctx* c, const Factor& f) {
  if (c->n_c == 0 || c->n_items == 0) return;
  SolveDev a = c->solve_dev;
  a.Linv = f.Linv;
  a.LR = f.LR;
  SC_CUDA(cudaMemsetAsync(c->d_solve_cnt, 0, sizeof(int) * (4 * (size_t)c->n_sn + 1), c->stream));
  const size_t smem = sizeof(double) * std::max(1, c->max_w);
  static int attr_set = 0;
  if (!attr_set) {
    SC_CUDA(cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(48 * 1024)));
    attr_set = 1;
  }
  if (c->solve_grid == 0) {
    int per_sm = 0, sms = 0, dev = 0;
    SC_CUDA(cudaGetDevice(&dev));
    SC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve, 256, smem));
    c->solve_grid = std::max(1, std::min(c->n_items, per_sm * sms));
  }
  k_solve<<<c->solve_grid, 256, smem, c->stream>>>(a);
  SC_CUDA(cudaGetLastError());
}
