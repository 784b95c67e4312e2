// Per-step kernels of libsc: one Newmark IMEX step:
//  (a1)+(a2)  k_explicit_{1,2,3}d : r^d = -K^d u_n on the all-uncut lattice (tensor form,
//             assembled 1D operators, sum factorised) fused with the CDM sum step
//             u^d_{n+1} = 2u^d_n - u^d_{n-1} + dt^2 r^d / M^dd
//  (a1)+(a2)  k_irregular : the same for d DOFs touching an empty cell or carrying f_x
//  (a3)+(a4)  k_celem     : predictor u~^c fused into the element products K_e w_e of the
//             c elements (dense cut K_e, reference uncut K_e);  k_crhs gathers
//             r^c = f_t(t_{n+1}) f_x^c - (K w)_c
//  (a5)       k_fwdA/k_fwdB/k_bwdA/k_bwdB : supernodal triangular solves with L_ss^{-1}
//  (a6)       k_corrector
// Buffers: d_u[cur] = u_n (lattice, holes = 0), d_u[cur^1] = u_{n-1} on d nodes; the step
// writes u_{n+1} into d_u[cur^1] (d nodes by (a2), c nodes by (a6)) and flips cur.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "sc_internal.h"

#include "explicit_common.cuh"

namespace {

__device__ __forceinline__ double wt(int i, int e_cnt, int P) {
  // assembled 1D GLL weight of lattice node i (N elements of order P)
  const int l = i % P, e = i / P;
  if (l) return c_w[l];
  return (e > 0 ? c_w[P] : 0.0) + (e < e_cnt ? c_w[0] : 0.0);
}

// assembled 1D operator A (c_Mh or c_Kh) applied at node gi; v(k) returns the value at
// global index k.  Sums over the (1 or 2) incident elements inside [0, Ne).
template <int P, typename F>
__device__ __forceinline__ double op1d(const double* A, int gi, int Ne, F v) {
  const int e = gi / P, l = gi - e * P;
  double s = 0.0;
  if (l) {
#pragma unroll
    for (int k = 0; k <= P; ++k) s += A[l * (P + 1) + k] * v(e * P + k);
    return s;
  }
  if (e > 0) {
#pragma unroll
    for (int k = 0; k <= P; ++k) s += A[P * (P + 1) + k] * v((e - 1) * P + k);
  }
  if (e < Ne) {
#pragma unroll
    for (int k = 0; k <= P; ++k) s += A[k] * v(e * P + k);
  }
  return s;
}

// ------------------------------------------------------------------ 1D
template <int P>
__global__ void k_explicit_1d(const double* __restrict__ U, const double* Pv, double* out,
                              const uint8_t* __restrict__ nt, ExpP e, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.nl[0] || !((e.want >> nt[i]) & 1)) return;
  const double r = e.s[0] * op1d<P>(c_Kh, i, e.N[0], [&](int k) { return U[k]; });
  const double u = U[i];
  const double res = e.a1 * u + e.a2 * Pv[i] - e.coefR * r / wt(i, e.N[0], P);
  out[i] = res;
  if (!isfinite(res)) atomicExch(flag, 1);
}

#include "explicit3d.cuh"
#include "explicit3d_v2.cuh"
#include "explicit2d.cuh"

// ------------------------------------------------------------------ irregular d nodes
__device__ __forceinline__ double ft_at(const double* ft, long long nt_, const long long* step, int off) {
  const long long n = *step + off;
  return (n >= 0 && n < nt_) ? ft[n] : 0.0;
}

__global__ void k_irregular(const double* __restrict__ U, const double* Pv, double* out, const int32_t* __restrict__ lat,
                            const double* __restrict__ invm, const double* __restrict__ fx, int n,
                            const int8_t* __restrict__ cls, const double* __restrict__ Kref, GridP g,
                            const double* __restrict__ ft, long long n_t, const long long* step, double a1,
                            double a2, double a3, int* flag, double fsc) {
  // one warp per node; lanes split the element-local dot products (fsc scales the load term)
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= n) return;
  const long long L = lat[t];
  const int P = g.p, n1 = P + 1;
  int nb = n1;
  if (g.dim > 1) nb *= n1;
  if (g.dim > 2) nb *= n1;
  long long ijk[3];
  long long rem = L;
  int e0[3], e1[3];
  for (int k = 0; k < 3; ++k) {
    if (k < g.dim) {
      ijk[k] = rem % g.nl[k];
      rem /= g.nl[k];
      if (ijk[k] % P == 0) {
        e0[k] = (int)(ijk[k] / P) - 1;
        e1[k] = (int)(ijk[k] / P);
      } else {
        e0[k] = e1[k] = (int)(ijk[k] / P);
      }
      if (e0[k] < 0) e0[k] = e1[k];
      if (e1[k] >= g.N[k]) e1[k] = e0[k];
    } else {
      ijk[k] = 0;
      e0[k] = e1[k] = 0;
    }
  }
  double Ku = 0.0;
  for (int c2 = e0[2]; c2 <= e1[2]; ++c2)
    for (int c1 = e0[1]; c1 <= e1[1]; ++c1)
      for (int c0 = e0[0]; c0 <= e1[0]; ++c0) {
        const long long ci = c0 + (long long)g.N[0] * (c1 + (long long)(g.dim > 1 ? g.N[1] : 1) * c2);
        if (cls[ci] == 2) continue;
        const int cc[3] = {c0, c1, c2};
        int li = 0, mul = 1;
        for (int k = 0; k < g.dim; ++k) {
          li += (int)(ijk[k] - (long long)cc[k] * P) * mul;
          mul *= n1;
        }
        for (int loc = lane; loc < nb; loc += 32) {
          const int l0 = loc % n1, l1 = (loc / n1) % n1, l2 = loc / (n1 * n1);
          long long gl = (long long)c0 * P + l0;
          if (g.dim > 1) gl += g.nl[0] * ((long long)c1 * P + l1);
          if (g.dim > 2) gl += g.nl[0] * g.nl[1] * ((long long)c2 * P + l2);
          Ku += Kref[(size_t)li * nb + loc] * U[gl];
        }
      }
#pragma unroll
  for (int o = 16; o; o >>= 1) Ku += __shfl_xor_sync(0xffffffffu, Ku, o);
  if (lane) return;
  const double r = fsc * ft_at(ft, n_t, step, 0) * fx[t] - Ku;
  const double res = a1 * U[L] + a2 * Pv[L] + a3 * r * invm[t];
  out[L] = res;
  if (!isfinite(res)) atomicExch(flag, 1);
}

// distributed load on tensor-d nodes (source kind 2): the explicit kernel has written
// a1 u + a2 Pv - a3 (K u)/M; add a3 f_t(t_n) f_x / M (eq:CDMacc)
__global__ void k_load_d(double* __restrict__ out, const int32_t* __restrict__ lat, const double* __restrict__ fxm,
                         int n, const double* __restrict__ ft, long long n_t, const long long* step, double a3) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[lat[i]] += a3 * ft_at(ft, n_t, step, 0) * fxm[i];
}

static void launch_load_d(sc_ctx* c, double* out, double a3, cudaStream_t st) {
  if (c->n_load == 0) return;
  k_load_d<<<(unsigned)((c->n_load + 255) / 256), 256, 0, st>>>(out, c->d_load_lat, c->d_load_fxm, (int)c->n_load,
                                                                c->d_ft, c->n_t, c->d_step, a3);
  SC_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ c elements
// mode 0 (step): w = predictor u~^c on c nodes, u^d_{n+1} (buffer B) elsewhere;
// mode 1 (start): w = A everywhere;
// mode 2 (leap-frog substep, integrator 4): w = u^c_k (compact, vc) on c nodes, the d values
// A + theta (B - A) elsewhere (reading LF3: theta = k/m interpolated, 0 frozen).
// Y[e][i] = sum_j K_e[i][j] w_j (K_e symmetric: read as columns, coalesced across threads).
// k_celem streams a dense K_e (element sizes without a packed kernel); cut elements of the
// common sizes use k_celem_sym on the packed lower triangle (below).
#ifndef CELEM_U
#define CELEM_U 8
#endif
#ifndef CELEM_CS
#define CELEM_CS 0
#endif
#ifndef CESYM_PF
#define CESYM_PF 0
#endif
#ifndef CESYM_OFF
#define CESYM_OFF 0
#endif
#ifndef CESYM_G
#define CESYM_G 8
#endif
__host__ __device__ constexpr int brev5(int n) {
  return ((n & 1) << 4) | ((n & 2) << 2) | (n & 4) | ((n & 8) >> 2) | ((n & 16) >> 4);
}
// local node j of c element e: its value in w_e = [u^d_{n+1}; u~^c] (mode 0: predictor for c
// nodes), u (mode 1), or the leap-frog substep value (mode 2)
__device__ __forceinline__ double celem_w(int mode, const double* __restrict__ A, const double* __restrict__ B,
                                          const double* __restrict__ vc, const double* __restrict__ ac, double dt,
                                          const int32_t* __restrict__ ecidx, int e, int nb, int j,
                                          const long long ci[3], const GridP& g, double theta) {
  const int n1 = g.p + 1;
  const int l0 = j % n1, l1 = (j / n1) % n1, l2 = j / (n1 * n1);
  long long gl = ci[0] * g.p + l0;
  if (g.dim > 1) gl += g.nl[0] * (ci[1] * g.p + l1);
  if (g.dim > 2) gl += g.nl[0] * g.nl[1] * (ci[2] * g.p + l2);
  if (mode == 1) return A[gl];
  const int cc = ecidx[(size_t)e * nb + j];
  if (mode == 2) return cc >= 0 ? vc[cc] : fma(theta, B[gl] - A[gl], A[gl]);
  return cc >= 0 ? A[gl] + dt * vc[cc] + 0.25 * dt * dt * ac[cc] : B[gl];
}

__device__ __forceinline__ void cell_ci(const GridP& g, long long cell, long long ci[3]) {
  long long rem = cell;
  for (int k = 0; k < 3; ++k) {
    if (k < g.dim) {
      ci[k] = rem % g.N[k];
      rem /= g.N[k];
    } else {
      ci[k] = 0;
    }
  }
}

// ids: the c elements of this launch (the cut ones: their dense K_e is streamed once)
__global__ void k_celem(int mode, const double* __restrict__ A, const double* __restrict__ B,
                        const double* __restrict__ vc, const double* __restrict__ ac, double dt,
                        const int32_t* __restrict__ ecell, const int32_t* __restrict__ ekidx,
                        const int32_t* __restrict__ ecidx, const double* __restrict__ Kcut,
                        const double* __restrict__ Kref, double* __restrict__ Y, int ne, int nb, int tpe, GridP g,
                        double theta, const int32_t* __restrict__ ids) {
  extern __shared__ double sw[];
  const int epb = blockDim.x / tpe;
  const int le = threadIdx.x / tpe, i = threadIdx.x % tpe;
  const int slot = blockIdx.x * epb + le;
  const bool ok = slot < ne;
  const int e = ok ? ids[slot] : 0;
  const int n1 = g.p + 1;
  double* w = sw + le * nb;
  if (ok) {
    long long ci[3];
    cell_ci(g, ecell[e], ci);
    for (int j = i; j < nb; j += tpe) w[j] = celem_w(mode, A, B, vc, ac, dt, ecidx, e, nb, j, ci, g, theta);
  }
  __syncthreads();
  if (!ok) return;
  const int kidx = ekidx[e];
  const double* K = kidx >= 0 ? Kcut + (size_t)kidx * nb * nb : Kref;
  auto gemv = [&](auto ld) {
    for (int r = i; r < nb; r += tpe) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      int j = 0;
      for (; j + CELEM_U <= nb; j += CELEM_U) {   // CELEM_U independent loads in flight (HBM-bound GEMV)
        double x[CELEM_U];
#pragma unroll
        for (int k = 0; k < CELEM_U; ++k) x[k] = ld(K + (size_t)(j + k) * nb + r);
#pragma unroll
        for (int k = 0; k < CELEM_U; ++k) acc[k & 3] += x[k] * w[j + k];
      }
      for (; j < nb; ++j) acc[0] += ld(K + (size_t)j * nb + r) * w[j];
      Y[(size_t)e * nb + r] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    }
  };
  // cut-cell matrices are streamed once per step (evict-first); the shared uncut reference
  // matrix stays cached
  if (CELEM_CS && kidx >= 0) gemv([](const double* p) { return __ldcs(p); });
  else gemv([](const double* p) { return __ldg(p); });
}

// Cut c elements on the PACKED lower triangle of their symmetric K_e (row i holds K[i][0..i]
// at offset i(i+1)/2: nb(nb+1)/2 doubles, 50.4% of the dense bytes at nb = 125).  One warp
// per element; lane l owns the columns j = l + 32c.  Row i is read coalesced (lanes over
// j <= i) and every stored entry is used twice:
//   row part     s_i   = sum_{j<=i} K_ij w_j   (per-lane partials, 32 rows per block, then
//                                                one transposing butterfly: lane m gets row m)
//   column part  t_j  += K_ij w_i  (j < i)     (lane-owned accumulators, no reduction)
// so y = s + t.  w_i is broadcast by a shuffle from its owning lane.  The row loop is
// unrolled at compile time (NB), so every load has an immediate offset from the element base.
#ifndef CESYM_MINB
#define CESYM_MINB 10
#endif
#if CESYM_MINB > 0
#define CESYM_LB __launch_bounds__(128, CESYM_MINB)
#else
#define CESYM_LB __launch_bounds__(128)
#endif
// L2 prefetch of packed rows [r0, r1) of the element (lanes over 128-byte lines)
__device__ __forceinline__ void cesym_prefetch(const double* K, int r0, int r1, int lane) {
  const char* a = (const char*)(K + (long long)r0 * (r0 + 1) / 2);
  const char* b = (const char*)(K + (long long)r1 * (r1 + 1) / 2);
  const char* a0 = (const char*)((unsigned long long)a & ~127ull);
  for (const char* q = a0 + 128 * lane; q < b; q += 128 * 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
}
template <int NB>
__global__ void CESYM_LB k_celem_sym(int mode, const double* __restrict__ A, const double* __restrict__ B,
                                                   const double* __restrict__ vc, const double* __restrict__ ac,
                                                   double dt, const int32_t* __restrict__ ecell,
                                                   const int32_t* __restrict__ ekidx, const int32_t* __restrict__ ecidx,
                                                   const double* __restrict__ Kpk, double* __restrict__ Y, int ne,
                                                   GridP g, double theta, const int32_t* __restrict__ ids) {
  constexpr int NK = (NB + 31) / 32;
  constexpr long long NT = (long long)NB * (NB + 1) / 2;
  const int lane = threadIdx.x & 31;
  const int slot = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (slot >= ne) return;   // warp-uniform
  const int e = ids[slot];
  const double* __restrict__ K = Kpk + (long long)ekidx[e] * NT;
#if CESYM_PF
  // the element's whole packed triangle as one bulk L2 prefetch (16-byte granules), issued
  // before the w gather so that the row loads below find it in L2
  if (lane == 0) {
    const unsigned long long a0 = (unsigned long long)K & ~15ull;
    const unsigned long long a1 = ((unsigned long long)(K + NT) + 15ull) & ~15ull;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
  }
#endif
#if CESYM_PF == 2
  cesym_prefetch(K, 0, NB < 64 ? NB : 64, lane);
#endif
  long long ci[3];
  cell_ci(g, ecell[e], ci);
  double wr[NK], at[NK], yr[NK];
#pragma unroll
  for (int c = 0; c < NK; ++c) {
    const int j = lane + 32 * c;
    wr[c] = j < NB ? celem_w(mode, A, B, vc, ac, dt, ecidx, e, NB, j, ci, g, theta) : 0.0;
    at[c] = 0.0;
  }
#pragma unroll
  for (int b = 0; b < NK; ++b) {
    // rows in bit-reversed order n -> m = brev5(n): the transposing butterfly (31 shuffles
    // per 32 rows) then runs as a binary counter over the row partials -- the stage of width
    // 16 >> lv pairs consecutive results of level lv -- so at most 5 partials stay live and
    // the registers go to loads in flight (CESYM_G rows' loads issued before their FMAs)
#if CESYM_PF == 2
    if (b >= 1 && 32 * (b + 1) < NB) cesym_prefetch(K, 32 * (b + 1), 32 * (b + 2) < NB ? 32 * (b + 2) : NB, lane);
#endif
    double pend[5], cur = 0.0;
#pragma unroll
    for (int n0 = 0; n0 < 32; n0 += CESYM_G) {
      double x[CESYM_G][NK];
#pragma unroll
      for (int gq = 0; gq < CESYM_G; ++gq) {
        const int m = brev5(n0 + gq), i = 32 * b + m;
#pragma unroll
        for (int c = 0; c <= b; ++c) {
          x[gq][c] = 0.0;
          if (i < NB && (c < b || lane <= m)) x[gq][c] = __ldg(K + i * (i + 1) / 2 + lane + 32 * c);   // j <= i
        }
      }
#pragma unroll
      for (int gq = 0; gq < CESYM_G; ++gq) {
        const int n = n0 + gq, m = brev5(n), i = 32 * b + m;
        double p = 0.0;
        if (i < NB) {
          const double wi = __shfl_sync(0xffffffffu, wr[b], m);
#pragma unroll
          for (int c = 0; c <= b; ++c) {
            p = fma(x[gq][c], wr[c], p);
            if (c < b || lane < m) at[c] = fma(x[gq][c], wi, at[c]);
          }
        }
        cur = p;
#pragma unroll
        for (int lv = 0; lv < 5; ++lv) {
          if (((n >> lv) & 1) == 0) {
            pend[lv] = cur;
            break;
          }
          // stage of width w: each lane keeps the partner whose row bit w matches its lane bit
          const int w = 16 >> lv;
          const bool up = (lane & w) != 0;
          const double lo = pend[lv], hi = cur;
          cur = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, w);
        }
      }
    }
    yr[b] = cur;   // n = 31 carried through all five levels: lane l holds row 32b + l
  }
#pragma unroll
  for (int c = 0; c < NK; ++c) {
    const int j = lane + 32 * c;
    if (j < NB) Y[(size_t)e * NB + j] = yr[c] + at[c];
  }
}

// setup: dense symmetric K_e -> packed lower triangle (one CTA per cut cell)
__global__ void k_pack_lower(const double* __restrict__ K, double* __restrict__ P, int nb) {
  const long long e = blockIdx.x;
  const long long nt = (long long)nb * (nb + 1) / 2;
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    int i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((long long)i * (i + 1) / 2 > t) --i;
    while ((long long)(i + 1) * (i + 2) / 2 <= t) ++i;
    const int j = t - i * (i + 1) / 2;
    P[e * nt + t] = K[(e * nb + i) * nb + j];
  }
}

// nb with a packed-symmetric cut-element kernel
static bool celem_sym_nb(int nb) {
  if (CESYM_OFF) return false;
  return nb == 125 || nb == 64 || nb == 27 || nb == 25 || nb == 5;
}

// Uncut c elements all share the reference K_e (Kref, symmetric): Y_e = Kref w_e for a batch of
// CR_EB elements is one small GEMM Kref [nb x nb] x W [nb x CR_EB].  W gathered into shared
// memory; each thread a 4-row x CR_EPW-element register tile (lanes over rows, warps over
// elements), Kref rows read through L1 (128 KB, cached), W broadcast from shared memory:
// per j, 4 row loads + CR_EPW/2 16-byte W loads feed 4 CR_EPW FMAs.  Every (row, element)
// sum runs over j in ascending order whatever the tile, so the result does not depend on
// CR_EPW / CR_NW (8-element tiles at 108 registers measured slower: the loop is
// latency-bound, profiles/r2_variants.txt).
#ifndef CR_EPW
#define CR_EPW 4    // elements per warp (8 measured slower: profiles/r2_variants.txt)
#endif
#ifndef CR_NW
#define CR_NW 8     // warps per CTA
#endif
#define CR_NT (32 * CR_NW)
#define CR_EB (CR_NW * CR_EPW)
template <int NB>   // nodes per element (compile time: the product loop is unrolled)
__global__ void __launch_bounds__(CR_NT) k_celem_ref(int mode, const double* __restrict__ A, const double* __restrict__ B,
                                                   const double* __restrict__ vc, const double* __restrict__ ac,
                                                   double dt, const int32_t* __restrict__ ecell,
                                                   const int32_t* __restrict__ ecidx, const double* __restrict__ Kref,
                                                   double* __restrict__ Y, int n, int /*nb*/, GridP g, double theta,
                                                   const int32_t* __restrict__ ids) {
  constexpr int nb = NB;
  extern __shared__ __align__(16) double sW[];   // [nb][CR_EB]
  __shared__ long long sci[CR_EB][3];
  __shared__ int se[CR_EB];
  const int s0 = blockIdx.x * CR_EB;
  const int ne = min(CR_EB, n - s0);
  if (threadIdx.x < ne) {   // cell coordinates once per element
    const int e = ids[s0 + threadIdx.x];
    se[threadIdx.x] = e;
    long long ci[3];
    cell_ci(g, ecell[e], ci);
    for (int k = 0; k < 3; ++k) sci[threadIdx.x][k] = ci[k];
  }
  __syncthreads();
  // gather W: GU entries per thread at a time in two passes, so that their loads are in flight
  // together (lattice index + c index first, then the values)
  constexpr int GT = CR_EB * 128 / CR_NT;   // entries per thread
  constexpr int GU = GT < 16 ? GT : 16;
  static_assert(GT % GU == 0, "gather chunks");
  const int n1 = g.p + 1;
  for (int u0 = 0; u0 < GT; u0 += GU) {
    long long glv[GU];
    int ccv[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      const int t = threadIdx.x + (u0 + u) * CR_NT;
      const int b = t / nb, j = t - b * nb;
      glv[u] = -1;
      ccv[u] = -1;
      if (t < CR_EB * nb && b < ne) {
        const int l0 = j % n1, l1 = (j / n1) % n1, l2 = j / (n1 * n1);
        long long gl = sci[b][0] * g.p + l0;
        if (g.dim > 1) gl += g.nl[0] * (sci[b][1] * g.p + l1);
        if (g.dim > 2) gl += g.nl[0] * g.nl[1] * (sci[b][2] * g.p + l2);
        glv[u] = gl;
        if (mode != 1) ccv[u] = ecidx[(size_t)se[b] * nb + j];
      }
    }
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      const int t = threadIdx.x + (u0 + u) * CR_NT;
      if (t >= CR_EB * nb) break;
      const int b = t / nb, j = t - b * nb;
      double v = 0.0;
      const long long gl = glv[u];
      const int cc = ccv[u];
      if (gl >= 0) {
        if (mode == 1) v = A[gl];
        else if (mode == 2) v = cc >= 0 ? vc[cc] : fma(theta, B[gl] - A[gl], A[gl]);
        else v = cc >= 0 ? A[gl] + dt * vc[cc] + 0.25 * dt * dt * ac[cc] : B[gl];
      }
      sW[j * CR_EB + b] = v;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wg = threadIdx.x >> 5;
  const int b0 = wg * CR_EPW;   // this warp's elements; lanes take rows lane + 32 a (coalesced)
  if (b0 >= ne) return;
  for (int rb = 0; rb < nb; rb += 128) {   // nb <= 128 in 3D p = 4: one pass
    double acc[4][CR_EPW];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < CR_EPW; ++c) acc[a][c] = 0.0;
#pragma unroll 5
    for (int j = 0; j < nb; ++j) {
      double k[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int r = rb + lane + 32 * a;
        k[a] = r < nb ? __ldg(Kref + (size_t)j * nb + r) : 0.0;   // Kref[r][j] (symmetric)
      }
      const double* wj = sW + j * CR_EB + b0;
      double w[CR_EPW];
#pragma unroll
      for (int c = 0; c < CR_EPW; c += 2) {
        const double2 w2 = *reinterpret_cast<const double2*>(wj + c);
        w[c] = w2.x;
        w[c + 1] = w2.y;
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < CR_EPW; ++c) acc[a][c] = fma(k[a], w[c], acc[a][c]);
    }
#pragma unroll
    for (int c = 0; c < CR_EPW; ++c) {
      if (b0 + c >= ne) break;
      double* y = Y + (size_t)se[b0 + c] * nb;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int r = rb + lane + 32 * a;
        if (r < nb) y[r] = acc[a][c];
      }
    }
  }
}

__global__ void k_crhs(double* __restrict__ b, const double* __restrict__ fxc, const int32_t* __restrict__ ptr,
                       const int32_t* __restrict__ idx, const double* __restrict__ Y, int nc,
                       const double* __restrict__ ft, long long n_t, const long long* step, int off,
                       const double* __restrict__ dscale, double fsc = 1.0, double theta = 0.0) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  double s = 0.0;
  for (int q = ptr[i]; q < ptr[i + 1]; ++q) s += Y[idx[q]];
  // f_t at t_{n+off} (+ theta dt: linear interpolation of the samples, leap-frog reading LF4)
  const double f0 = ft_at(ft, n_t, step, off);
  const double ftv = theta == 0.0 ? f0 : (1.0 - theta) * f0 + theta * ft_at(ft, n_t, step, off + 1);
  const double r = fsc * ftv * fxc[i] - s;
  b[i] = dscale ? dscale[i] * r : r;   // D r^c (scaled system) or r^c
}

// CDM on the c DOFs with the HRZ-lumped mass (integrator 1): u^c_{n+1} = 2u^c_n - u^c_{n-1}
// + dt^2 r^c / m^c, r^c = f_t(t_n) f_x^c - (K u_n)_c (P:577, P:580-583 with M~ of P:604-611)
__global__ void k_cdm_c(const double* __restrict__ A, double* __restrict__ B, const double* __restrict__ r,
                        const double* __restrict__ mc, const int32_t* __restrict__ clat, int nc, double dt2,
                        int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  const int32_t L = clat[i];
  const double un = 2.0 * A[L] - B[L] + dt2 * r[i] / mc[i];
  B[L] = un;
  if (!isfinite(un)) atomicExch(flag, 1);
}

// CDM on the consistent SCM at the c DOFs (integrator 3): u^c_{n+1} = 2u^c_n - u^c_{n-1} +
// dt^2 a^c_n with M^cc a^c_n = r^c (the solve returns x with a = D x, Jacobi scaling)
__global__ void k_cdm_cons(const double* __restrict__ A, double* __restrict__ B, const double* __restrict__ x,
                           const double* __restrict__ dscale, const int32_t* __restrict__ clat, int nc, double dt2,
                           int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  const int32_t L = clat[i];
  const double un = 2.0 * A[L] - B[L] + dt2 * (dscale[i] * x[i]);
  B[L] = un;
  if (!isfinite(un)) atomicExch(flag, 1);
}

// start of integrator 3 at the c DOFs: u_{-1} = u_0 - dt v_0 + dt^2/2 a_0 (a_0 = D x, M solve)
__global__ void k_start_cons(const double* __restrict__ A, double* __restrict__ B, const double* __restrict__ x,
                             const double* __restrict__ dscale, const double* __restrict__ vlat,
                             const int32_t* __restrict__ clat, int nc, double dt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  const int32_t L = clat[i];
  B[L] = A[L] - (vlat ? dt * vlat[L] : 0.0) + 0.5 * dt * dt * (dscale[i] * x[i]);
}

// start of integrator 1 at the c DOFs: u_{-1} = u_0 - dt v_0 + dt^2/2 a_0, a_0 = r^c / m^c
__global__ void k_start_hrz(const double* __restrict__ A, double* __restrict__ B, const double* __restrict__ r,
                            const double* __restrict__ mc, const double* __restrict__ vlat,
                            const int32_t* __restrict__ clat, int nc, double dt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  const int32_t L = clat[i];
  B[L] = A[L] - (vlat ? dt * vlat[L] : 0.0) + 0.5 * dt * dt * r[i] / mc[i];
}

// leap-frog substep of the c DOFs (integrator 4, reading LF2): u^c_{k+1} = 2u^c_k - u^c_{k-1}
// + dt_f^2 a_k with M^cc a_k = r^c (the solve returns x, a = D x); uc = u^c_k, up = u^c_{k-1}
__global__ void k_lf_sub(double* __restrict__ uc, double* __restrict__ up, const double* __restrict__ x,
                         const double* __restrict__ dscale, int nc, double dtf2, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  const double cur = uc[i];
  const double un = 2.0 * cur - up[i] + dtf2 * (dscale[i] * x[i]);
  up[i] = cur;
  uc[i] = un;
  if (!isfinite(un)) atomicExch(flag, 1);
}
// u^c_{n+1} into the lattice buffer
__global__ void k_lf_store(const double* __restrict__ uc, double* __restrict__ B, const int32_t* __restrict__ clat,
                           int nc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nc) B[clat[i]] = uc[i];
}
// start of integrator 4 at the c DOFs (fine level): u^c_0 and u^c_{-1} = u^c_0 - dt_f v_0 +
// dt_f^2/2 a_0 (a_0 = D x from the M solve of the start)
__global__ void k_start_lf(const double* __restrict__ A, double* __restrict__ uc, double* __restrict__ up,
                           const double* __restrict__ x, const double* __restrict__ dscale,
                           const double* __restrict__ vlat, const int32_t* __restrict__ clat, int nc, double dtf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  const int32_t L = clat[i];
  uc[i] = A[L];
  up[i] = A[L] - (vlat ? dtf * vlat[L] : 0.0) + 0.5 * dtf * dtf * (dscale[i] * x[i]);
}

// M^{-1} K x at the c DOFs with the consistent M^cc (power iteration of integrator 3):
// the M solve of r = -(K x)_c returned a = D x
__global__ void k_cons_apply(double* __restrict__ Y, const double* __restrict__ x, const double* __restrict__ dscale,
                             const int32_t* __restrict__ clat, int nc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nc) Y[clat[i]] = -dscale[i] * x[i];
}

// M~^{-1} K x at the c DOFs (power iteration of integrator 1): r = -(K x)_c
__global__ void k_hrz_apply(double* __restrict__ Y, const double* __restrict__ r, const double* __restrict__ mc,
                            const int32_t* __restrict__ clat, int nc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nc) Y[clat[i]] = -r[i] / mc[i];
}

// ------------------------------------------------------------------ corrector / misc
__global__ void k_corrector(const double* __restrict__ A, double* __restrict__ B, double* __restrict__ vc,
                            double* __restrict__ ac, const double* __restrict__ x, const int32_t* __restrict__ clat,
                            int nc, double dt, int* flag, const double* __restrict__ dscale) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  const int32_t L = clat[i];
  const double v = vc[i], a = ac[i];
  const double ut = A[L] + dt * v + 0.25 * dt * dt * a;   // (a3) predictor
  const double vt = v + 0.5 * dt * a;
  const double an = dscale[i] * x[i];                      // (a5) result, x = D y
  const double un = ut + 0.25 * dt * dt * an;              // (a6) corrector
  B[L] = un;
  vc[i] = vt + 0.5 * dt * an;
  ac[i] = an;
  if (!isfinite(un)) atomicExch(flag, 1);
}

__global__ void k_start_c(double* __restrict__ ac, double* __restrict__ vc, const double* __restrict__ x,
                          const double* __restrict__ vlat, const int32_t* __restrict__ clat, int nc,
                          const double* __restrict__ dscale) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  ac[i] = dscale[i] * x[i];
  vc[i] = vlat ? vlat[clat[i]] : 0.0;
}

__global__ void k_advance(long long* step) { *step += 1; }

// receivers: row *step of the trace = sum_k w[r][k] u[lat[r][k]] (warp per receiver)
__global__ void k_record(const double* __restrict__ u, const int32_t* __restrict__ lat,
                         const double* __restrict__ w, int n_rec, int nb, double* trace, long long cap,
                         const long long* step) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const long long row = *step;
  if (r >= n_rec || row >= cap) return;
  double s = 0.0;
  for (int k = lane; k < nb; k += 32) s += w[(size_t)r * nb + k] * u[lat[(size_t)r * nb + k]];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) trace[row * n_rec + r] = s;
}

__global__ void k_gather(const double* __restrict__ lat, const int64_t* __restrict__ idx, double* __restrict__ out,
                         long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = lat[idx[i]];
}

__global__ void k_scatter(const double* __restrict__ in, const int64_t* __restrict__ idx, double* __restrict__ lat,
                          long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) lat[idx[i]] = in[i];
}

// ------------------------------------------------------------------ launch helpers
template <int P> struct Tile2 { static constexpr int E = P <= 4 ? 8 : 4; };

// tile extents (elements) of the explicit kernel for this p / dim: ext[k] elements per tile
// along k, tg[k] tiles along k
template <int P>
void tiling_p(const GridP& g, int ext[3], int tg[3]) {
  ext[0] = ext[1] = ext[2] = 1;
  if (g.dim == 2) {
    ext[0] = ext[1] = Tile2v<P>::E;
  } else if (g.dim == 3) {
    if constexpr (P <= 6) {
      ext[0] = Tile3<P>::E;
      ext[1] = Tile3<P>::EY;
      ext[2] = g.ezl > 0 ? g.ezl : Tile3<P>::EZ;
    }
  }
  for (int k = 0; k < 3; ++k) tg[k] = (g.N[k] + ext[k] - 1) / ext[k];
}

template <int P>
void launch_explicit_p(sc_ctx* c, const double* U, const double* Pv, double* out, ExpP e, int n_tiles,
                       int cap, cudaStream_t st) {
  const GridP& g = c->g;
  int ext[3], tg[3];
  tiling_p<P>(g, ext, tg);
  e.tg[0] = tg[0];
  e.tg[1] = tg[1];
  e.ezl = ext[2];
  e.ntiles = e.tiles ? n_tiles : tg[0] * tg[1] * tg[2];
  if (e.ntiles == 0) return;
  static int sms = 0;
  if (!sms) SC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  // cap > 0: at most cap resident CTAs per SM (grid-stride over the tiles)
  const unsigned grid = (unsigned)(cap > 0 ? std::min(e.ntiles, cap * sms) : e.ntiles);
  if (g.dim == 1) {
    k_explicit_1d<P><<<(unsigned)((g.nl[0] + 255) / 256), 256, 0, st>>>(U, Pv, out, c->d_ntype, e, c->d_flag);
  } else if (g.dim == 2) {
    constexpr int E2 = Tile2v<P>::E;
    k_explicit_2d<P, E2, E2, Tile2v<P>::NT><<<grid, Tile2v<P>::NT, 0, st>>>(U, Pv, out, c->d_ntype, e, c->d_flag);
  } else {
    if constexpr (P <= 6) {
      using T = Tile3<P>;
      // the shared-memory opt-in was set on this context's device at setup (explicit_prepare)
      v2::k_exp3<P, T::E, T::EY, T::NT, T::MINB><<<grid, T::NT, v2::smem3<P, T::E, T::EY>(), st>>>(U, Pv, out, c->d_ntype, e,
                                                                                       c->d_flag);
    }
  }
}

// per-context (per-device) kernel attributes, set at setup before any graph capture: the 3D
// explicit kernel's dynamic shared memory opt-in (~97 KB at p = 4)
template <int P>
void explicit_prepare_p(sc_ctx* c) {
  if constexpr (P <= 6) {
    using T = Tile3<P>;
    SC_CUDA(cudaFuncSetAttribute(v2::k_exp3<P, T::E, T::EY, T::NT, T::MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)v2::smem3<P, T::E, T::EY>()));
  }
  (void)c;
}

}  // namespace

void explicit_prepare(sc_ctx* c) {
  if (c->g.dim != 3) return;
  SC_CUDA(cudaSetDevice(c->device));
  switch (c->g.p) {
    case 1: explicit_prepare_p<1>(c); break;
    case 2: explicit_prepare_p<2>(c); break;
    case 3: explicit_prepare_p<3>(c); break;
    case 4: explicit_prepare_p<4>(c); break;
    case 5: explicit_prepare_p<5>(c); break;
    case 6: explicit_prepare_p<6>(c); break;
    default: break;
  }
}

void explicit_tiling(const GridP& g, int ext[3], int tg[3]) {
  switch (g.p) {
    case 1: tiling_p<1>(g, ext, tg); break;
    case 2: tiling_p<2>(g, ext, tg); break;
    case 3: tiling_p<3>(g, ext, tg); break;
    case 4: tiling_p<4>(g, ext, tg); break;
    case 5: tiling_p<5>(g, ext, tg); break;
    case 6: tiling_p<6>(g, ext, tg); break;
    case 7: tiling_p<7>(g, ext, tg); break;
    case 8: tiling_p<8>(g, ext, tg); break;
    default: throw ScError(SC_ERR_CONFIG, "p out of range");
  }
}

// (a1)+(a2) on the lattice nodes of type `want` (1: tensor-d far from c nodes, 4: tensor-d
// sharing an element with a c node).  want 4 runs over the near-tile list only.
void launch_explicit(sc_ctx* c, const double* U, const double* Pv, double* out, double a1, double a2, double a3,
                     int want, cudaStream_t st, int cap = 0) {
  const GridP& g = c->g;
  ExpP e;
  for (int k = 0; k < 3; ++k) {
    e.nl[k] = (int)g.nl[k];
    e.N[k] = g.N[k];
    e.s[k] = k < g.dim ? (2.0 / g.h[k]) * (2.0 / g.h[k]) : 0.0;
  }
  e.a1 = a1;
  e.a2 = a2;
  e.coefR = a3 * c->c * c->c;
  if (c->n_d == c->n_irr) return;   // no tensor-d DOFs (e.g. integrator 2: all implicit)
  e.want = want == 1 ? WANT_FAR : (want == 4 ? WANT_NEAR : WANT_FAR | WANT_NEAR);
  e.clean = want == 5 ? c->d_clean : nullptr;
  e.tiles = nullptr;
  int n_tiles = 0;
  if (want == 5 && c->n_near == 0) e.want = WANT_FAR;
  if (want == 4) {
    if (c->n_near == 0) return;
    if (g.dim > 1) {
      e.tiles = c->d_near_tiles;
      n_tiles = c->n_near_tiles;
    }
  } else if (c->world > 1 && g.dim > 1) {
    e.tiles = c->d_far_tiles;   // the tiles of this rank's region (they hold its near nodes too)
    n_tiles = c->n_far_tiles;
  }
  switch (g.p) {
    case 1: launch_explicit_p<1>(c, U, Pv, out, e, n_tiles, cap, st); break;
    case 2: launch_explicit_p<2>(c, U, Pv, out, e, n_tiles, cap, st); break;
    case 3: launch_explicit_p<3>(c, U, Pv, out, e, n_tiles, cap, st); break;
    case 4: launch_explicit_p<4>(c, U, Pv, out, e, n_tiles, cap, st); break;
    case 5: launch_explicit_p<5>(c, U, Pv, out, e, n_tiles, cap, st); break;
    case 6: launch_explicit_p<6>(c, U, Pv, out, e, n_tiles, cap, st); break;
    case 7: launch_explicit_p<7>(c, U, Pv, out, e, n_tiles, cap, st); break;
    case 8: launch_explicit_p<8>(c, U, Pv, out, e, n_tiles, cap, st); break;
    default: throw ScError(SC_ERR_CONFIG, "p out of range");
  }
  SC_CUDA(cudaGetLastError());
}

static void launch_celem(sc_ctx* c, int mode, const double* A, const double* B, cudaStream_t st,
                         double theta = 0.0, const double* vc = nullptr) {
  if (c->n_celem == 0) return;
  const int nb = c->nb;
  const int tpe = std::min(256, ((nb + 31) / 32) * 32);
  const int epb = 256 / tpe;
  const double* vcp = vc ? vc : c->d_vc;
  // the reference-element products run on a side stream beside the (HBM-bound) cut-element
  // stream: disjoint outputs, both only read the state; joined before returning
  const bool fork = c->n_celem_cut > 0 && c->n_celem_ref > 0;
  cudaStream_t sr = st;
  if (fork) {
    if (!c->s_ref) {
      SC_CUDA(cudaStreamCreateWithFlags(&c->s_ref, cudaStreamNonBlocking));
      SC_CUDA(cudaEventCreateWithFlags(&c->ev_ref0, cudaEventDisableTiming));
      SC_CUDA(cudaEventCreateWithFlags(&c->ev_ref1, cudaEventDisableTiming));
    }
    SC_CUDA(cudaEventRecord(c->ev_ref0, st));
    SC_CUDA(cudaStreamWaitEvent(c->s_ref, c->ev_ref0, 0));
    sr = c->s_ref;
  }
  if (c->n_celem_ref > 0) {
    const unsigned rb = (unsigned)((c->n_celem_ref + CR_EB - 1) / CR_EB);
    const size_t rsm = sizeof(double) * CR_EB * nb;
    auto ref = [&](auto kern) {
      kern<<<rb, CR_NT, rsm, sr>>>(mode, A, B, vcp, c->d_ac, c->dt, c->d_celem_cell, c->d_celem_cidx, c->d_Kref, c->d_Y,
                                 (int)c->n_celem_ref, nb, c->g, theta, c->d_celem_ref_ids);
    };
    if (nb == 125) {
      ref(k_celem_ref<125>);
    } else if (nb == 64) {
      ref(k_celem_ref<64>);
    } else if (nb == 27) {
      ref(k_celem_ref<27>);
    } else {   // other element sizes (2D, p >= 5 in 3D): the streaming kernel
      const unsigned blocks = (unsigned)((c->n_celem_ref + epb - 1) / epb);
      k_celem<<<blocks, epb * tpe, sizeof(double) * epb * nb, sr>>>(
          mode, A, B, vcp, c->d_ac, c->dt, c->d_celem_cell, c->d_celem_kidx, c->d_celem_cidx, c->d_Kcut, c->d_Kref,
          c->d_Y, (int)c->n_celem_ref, nb, tpe, c->g, theta, c->d_celem_ref_ids);
    }
    SC_CUDA(cudaGetLastError());
  }
  if (c->n_celem_cut > 0 && c->d_Kpk) {
    const unsigned blocks = (unsigned)((c->n_celem_cut + 3) / 4);
    auto sym = [&](auto kern) {
      kern<<<blocks, 128, 0, st>>>(mode, A, B, vcp, c->d_ac, c->dt, c->d_celem_cell, c->d_celem_kidx, c->d_celem_cidx,
                                   c->d_Kpk, c->d_Y, (int)c->n_celem_cut, c->g, theta, c->d_celem_cut_ids);
    };
    switch (nb) {
      case 125: sym(k_celem_sym<125>); break;
      case 64: sym(k_celem_sym<64>); break;
      case 27: sym(k_celem_sym<27>); break;
      case 25: sym(k_celem_sym<25>); break;
      case 5: sym(k_celem_sym<5>); break;
      default: throw ScError(SC_ERR_CONFIG, "packed K_e without a kernel");
    }
    SC_CUDA(cudaGetLastError());
  } else if (c->n_celem_cut > 0) {
    const unsigned blocks = (unsigned)((c->n_celem_cut + epb - 1) / epb);
    k_celem<<<blocks, epb * tpe, sizeof(double) * epb * nb, st>>>(
        mode, A, B, vcp, c->d_ac, c->dt, c->d_celem_cell, c->d_celem_kidx, c->d_celem_cidx, c->d_Kcut, c->d_Kref,
        c->d_Y, (int)c->n_celem_cut, nb, tpe, c->g, theta, c->d_celem_cut_ids);
    SC_CUDA(cudaGetLastError());
  }
  if (fork) {
    SC_CUDA(cudaEventRecord(c->ev_ref1, sr));
    SC_CUDA(cudaStreamWaitEvent(st, c->ev_ref1, 0));
  }
}

static void launch_irregular(sc_ctx* c, const double* U, const double* Pv, double* out, double a1, double a2,
                             double a3, cudaStream_t st, double fsc = 1.0) {
  if (c->n_irr == 0) return;
  k_irregular<<<(unsigned)((c->n_irr * 32 + 127) / 128), 128, 0, st>>>(
      U, Pv, out, c->d_irr_lat, c->d_irr_invm, c->d_irr_fx, (int)c->n_irr, c->d_cell_class, c->d_Kref, c->g,
      c->d_ft, c->n_t, c->d_step, a1, a2, a3, c->d_flag, fsc);
  SC_CUDA(cudaGetLastError());
}

// (a3)-(a6) of one step on stream st: predictor fused into the c-element products, r^c,
// the implicit solve S a^c_{n+1} = r^c, the corrector; then the device step counter.
static void enqueue_c_part(sc_ctx* c, const double* A, double* B, cudaStream_t st) {
  const double dt = c->dt;
  if (c->n_cl > 0 && c->integrator == 1) {
    // CDM with HRZ-lumped cut cells: (K u_n)_c from the c-element products, explicit update
    launch_celem(c, 1, A, A, st);
    k_crhs<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, st>>>(c->d_b, c->d_fxc, c->d_rhs_ptr, c->d_rhs_idx, c->d_Y,
                                                              (int)c->n_cl, c->d_ft, c->n_t, c->d_step, 0, nullptr);
    k_cdm_c<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, st>>>(A, B, c->d_b, c->d_mc, c->d_c_lat, (int)c->n_cl,
                                                               dt * dt, c->d_flag);
  } else if (c->n_cl > 0 && c->integrator == 4) {
    // leap-frog: m CDM substeps of the c DOFs with dt_f = dt/m on the consistent M^cc
    // (readings LF2-LF4); B already holds u^d_{n+1}; vc = u^c_k, ac = u^c_{k-1} (fine level)
    const int m = c->lf_m;
    const double dtf = dt / m;
    const unsigned gb = (unsigned)((c->n_cl + 255) / 256);
    for (int j = 0; j < m; ++j) {
      const double th = (double)j / m;
      launch_celem(c, 2, A, B, st, c->lf_coupling == 0 ? th : 0.0, c->d_vc);
      k_crhs<<<gb, 256, 0, st>>>(c->d_b, c->d_fxc, c->d_rhs_ptr, c->d_rhs_idx, c->d_Y, (int)c->n_cl, c->d_ft, c->n_t,
                                 c->d_step, 0, c->fM.d, 1.0, th);
      launch_solve(c, c->fM, st);
      k_lf_sub<<<gb, 256, 0, st>>>(c->d_vc, c->d_ac, c->d_x, c->fM.d, (int)c->n_cl, dtf * dtf, c->d_flag);
    }
    k_lf_store<<<gb, 256, 0, st>>>(c->d_vc, B, c->d_c_lat, (int)c->n_cl);
  } else if (c->n_cl > 0 && c->integrator == 3) {
    // CDM on the consistent SCM: M^cc a^c_n = f_t(t_n) f_x^c - (K u_n)_c with the M factor
    launch_celem(c, 1, A, A, st);
    k_crhs<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, st>>>(c->d_b, c->d_fxc, c->d_rhs_ptr, c->d_rhs_idx, c->d_Y,
                                                              (int)c->n_cl, c->d_ft, c->n_t, c->d_step, 0, c->fM.d);
    launch_solve(c, c->fM, st);
    k_cdm_cons<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, st>>>(A, B, c->d_x, c->fM.d, c->d_c_lat, (int)c->n_cl,
                                                                  dt * dt, c->d_flag);
  } else if (c->n_cl > 0) {
    launch_celem(c, 0, A, B, st);
    k_crhs<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, st>>>(c->d_b, c->d_fxc, c->d_rhs_ptr, c->d_rhs_idx, c->d_Y,
                                                              (int)c->n_cl, c->d_ft, c->n_t, c->d_step, 1, c->fS.d);
    if (!sc_knob("SC_DEBUG_NO_SOLVE")) launch_solve(c, c->fS, st);   // experiment builds only
    k_corrector<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, st>>>(A, B, c->d_vc, c->d_ac, c->d_x, c->d_c_lat,
                                                                  (int)c->n_cl, dt, c->d_flag, c->fS.d);
  }
  if (c->n_rec > 0)   // NEXT-3 observers: u at the receivers after this step
    k_record<<<(unsigned)((c->n_rec * 32 + 127) / 128), 128, 0, st>>>(B, c->d_rec_lat, c->d_rec_w, c->n_rec, c->nb,
                                                                        c->d_rec_trace, c->rec_cap, c->d_step);
  k_advance<<<1, 1, 0, st>>>(c->d_step);
  SC_CUDA(cudaGetLastError());
}

void destroy_graphs(sc_ctx* c) {
  for (int i = 0; i < 2; ++i)
    if (c->graph[i]) {
      cudaGraphExecDestroy(c->graph[i]);
      c->graph[i] = nullptr;
    }
}

// One Newmark IMEX step: u_n in d_u[parity], writes u_{n+1} into d_u[parity^1].
// Without c DOFs: the explicit update of every d node, then the step counter.
// With c DOFs the step is pipelined across steps: the far-d update of step
// n (type 1: no c node in any incident element) was already done by the previous graph;
// this graph does the near-d (type 4) and irregular updates of step n, then forks
//   stream s_hi (high priority): c part of step n  (reads u^c_n, u^d_{n+1}; writes u^c_{n+1})
//   stream st:                   far-d update of step n+1 (reads u_{n+1} at d nodes only,
//                                u_n at its own nodes; writes u_{n+2} at far-d nodes)
// which touch disjoint data, and joins them.
void enqueue_step(sc_ctx* c, int parity, cudaStream_t st) {
  double* A = c->d_u[parity];
  double* B = c->d_u[parity ^ 1];
  const double dt = c->dt;
  if (!c->pipelined) {
    // one explicit launch for far and near d nodes (want 5), irregular nodes, c part; with
    // world > 1 the pack of the exchange (the next step's explicit update needs it)
    launch_explicit(c, A, B, B, 2.0, -1.0, dt * dt, 5, st);
    launch_irregular(c, A, B, B, 2.0, -1.0, dt * dt, st);
    launch_load_d(c, B, dt * dt, st);
    enqueue_c_part(c, A, B, st);
    if (c->world > 1) enqueue_pack(c, B, st);
    return;
  }
  launch_explicit(c, A, B, B, 2.0, -1.0, dt * dt, 4, st);
  launch_irregular(c, A, B, B, 2.0, -1.0, dt * dt, st);
  SC_CUDA(cudaEventRecord(c->ev_fork, st));
  SC_CUDA(cudaStreamWaitEvent(c->s_hi, c->ev_fork, 0));
  enqueue_c_part(c, A, B, c->s_hi);
  SC_CUDA(cudaEventRecord(c->ev_join, c->s_hi));
  // far-d nodes of step n+1 on a capped grid: the c part keeps SM resources
  if (!sc_knob("SC_DEBUG_NO_FAR"))   // experiment builds only (wrong results when set)
    launch_explicit(c, B, A, A, 2.0, -1.0, dt * dt, 1, st, c->far_cap);
  SC_CUDA(cudaStreamWaitEvent(st, c->ev_join, 0));
}

// far-d update of the current step (type 1 nodes) when no previous graph did it
void enqueue_far_prologue(sc_ctx* c) {
  if (!c->pipelined || c->far_ready) return;
  const double* A = c->d_u[c->cur];
  double* B = c->d_u[c->cur ^ 1];
  launch_explicit(c, A, B, B, 2.0, -1.0, c->dt * c->dt, 1, c->stream);
  c->far_ready = true;
}

void build_graphs(sc_ctx* c) {
  // the far-d update of step n+1 is forked against the c part of step n; SC_FAR_CAP caps its
  // resident CTAs per SM and SC_SOLVE_CTAS_PER_SM those of the persistent solve (solve.cu) so
  // both can co-reside.  Measured on config 4 (profiles/): caps trade solve latency for
  // overlap one-for-one, so both default to the occupancy limit.
  if (const char* v = sc_knob("SC_FAR_CAP")) c->far_cap = std::max(0, atoi(v));
  // SC_PIPELINE=1: fork the far-d update of step n+1 against the c part of step n (one rank
  // with c DOFs); default off: measured no gain and it costs a second
  // (near-node) explicit launch
  c->pipelined = c->n_c > 0 && c->n_d > c->n_irr && c->world == 1 && c->integrator == 0 && c->n_load == 0 &&
                 sc_knob("SC_PIPELINE") &&
                 atoi(sc_knob("SC_PIPELINE"));
  if (!c->s_hi) {
    int lo = 0, hi = 0;
    SC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SC_CUDA(cudaStreamCreateWithPriority(&c->s_hi, cudaStreamNonBlocking, hi));
    SC_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    SC_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  }
  for (int par = 0; par < 2; ++par) {
    cudaGraph_t gr;
    SC_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    enqueue_step(c, par, c->stream);
    SC_CUDA(cudaStreamEndCapture(c->stream, &gr));
    // per-node priorities: the c part (captured on the high-priority stream) is dispatched ahead
    // of the concurrent far-d update
    SC_CUDA(cudaGraphInstantiate(&c->graph[par], gr, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(gr);
  }
  // kernels per step: explicit (+ near when pipelined) + irregular + advance + c part (+ pack)
  c->kernels_per_step = 1 + (c->pipelined && c->n_near > 0 ? 1 : 0) + (c->n_irr > 0) + (c->n_load > 0) + 1 +
                        (c->world > 1);
  if (c->n_c > 0)
    c->kernels_per_step += c->integrator == 1   ? 3
                           : c->integrator == 4 ? 4 * c->lf_m + 1
                                                : 3 + (c->n_items > 0 ? 1 : 0);
}

// near-d tile list: tiles of the explicit kernel that own at least one type-4 node (a tile
// owns nodes [ext*P*t, ext*P*(t+1)) per axis, the last tile also the final boundary node)
void setup_step_structures(sc_ctx* c) {
  GridP& g = c->g;
  explicit_prepare(c);
  // cut K_e -> packed lower triangles (the step streams half the bytes); the dense copy is
  // dropped once the host copy for the factorisation (setup_device_geometry) has landed
  if (c->n_cut > 0 && c->d_Kcut && celem_sym_nb(c->nb)) {
    const int nb = c->nb;
    SC_CUDA(cudaStreamSynchronize(c->stream));
    SC_CUDA(cudaMalloc(&c->d_Kpk, sizeof(double) * (size_t)c->n_cut * nb * (nb + 1) / 2));
    k_pack_lower<<<(unsigned)c->n_cut, 256, 0, c->stream>>>(c->d_Kcut, c->d_Kpk, nb);
    SC_CUDA(cudaGetLastError());
    SC_CUDA(cudaStreamSynchronize(c->stream));
    SC_CUDA(cudaFree(c->d_Kcut));
    c->d_Kcut = nullptr;
  }
  c->n_near_tiles = c->n_far_tiles = 0;
  if (g.dim == 1) return;
  int ext[3], tg[3];
  if (g.dim == 3) {
    // longer z tiles amortise the warm-up layer, but keep >= 4 waves of 2 CTAs per SM
    g.ezl = 16;
    explicit_tiling(g, ext, tg);
    if ((int64_t)tg[0] * tg[1] * tg[2] < 4 * 2 * 148) g.ezl = 8;
    if (const char* v = sc_knob("SC_EZL")) g.ezl = std::max(1, atoi(v));   // experiments
  }
  explicit_tiling(g, ext, tg);
  // tile lists of the node types this rank updates: near-d (type 4) always, far-d (type 1)
  // when world > 1 (the rank's region only)
  auto tiles_of = [&](unsigned want_mask, int** d, int* n) {
    std::vector<uint8_t> mark((size_t)tg[0] * tg[1] * tg[2], 0);
    for (int64_t L = 0; L < c->n_lat; ++L) {
      if (!((want_mask >> c->ntype_rank[L]) & 1)) continue;
      int64_t r = L;
      int64_t t[3] = {0, 0, 0};
      for (int k = 0; k < g.dim; ++k) {
        const int64_t i = r % g.nl[k];
        r /= g.nl[k];
        t[k] = std::min<int64_t>(i / ((int64_t)ext[k] * g.p), tg[k] - 1);
      }
      mark[t[0] + (size_t)tg[0] * (t[1] + (size_t)tg[1] * t[2])] = 1;
    }
    std::vector<int> tiles;
    for (size_t i = 0; i < mark.size(); ++i)
      if (mark[i]) tiles.push_back((int)i);
    *n = (int)tiles.size();
    SC_CUDA(cudaMalloc(d, sizeof(int) * std::max<size_t>(1, tiles.size())));
    if (!tiles.empty()) SC_CUDA(cudaMemcpy(*d, tiles.data(), sizeof(int) * tiles.size(), cudaMemcpyHostToDevice));
  };
  if (c->n_near) tiles_of(WANT_NEAR, &c->d_near_tiles, &c->n_near_tiles);
  // world > 1: the tiles holding this rank's tensor-d nodes, far OR near (the combined
  // launch updates both; a tile inside a void's c shell may hold near nodes only)
  if (c->world > 1) tiles_of(WANT_FAR | WANT_NEAR, &c->d_far_tiles, &c->n_far_tiles);
  // clean tiles (3D): every node a tile owns is tensor-d (type 1 or 4) -> the combined
  // far+near launch needs no per-node type loads there
  if (g.dim == 3) {
    const size_t nt_ = (size_t)tg[0] * tg[1] * tg[2];
    std::vector<uint8_t> clean(nt_, 1);
    for (int64_t L = 0; L < c->n_lat; ++L) {
      const uint8_t t = c->ntype_rank[L];
      if (t == 1 || t == 4) continue;
      int64_t r = L;
      int64_t ti[3] = {0, 0, 0};
      for (int k = 0; k < 3; ++k) {
        const int64_t i = r % g.nl[k];
        r /= g.nl[k];
        ti[k] = std::min<int64_t>(i / ((int64_t)ext[k] * g.p), tg[k] - 1);
      }
      clean[ti[0] + (size_t)tg[0] * (ti[1] + (size_t)tg[1] * ti[2])] = 0;
    }
    SC_CUDA(cudaMalloc(&c->d_clean, nt_));
    SC_CUDA(cudaMemcpy(c->d_clean, clean.data(), nt_, cudaMemcpyHostToDevice));
  }
}

// ---- multi-rank exchange (partition.cpp): pack this rank's values for all peers, unpack the
// received values (one buffer each, peers contiguous)
__global__ void k_pack(const double* __restrict__ u, const int32_t* __restrict__ idx, double* __restrict__ buf,
                       long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) buf[i] = u[idx[i]];
}
__global__ void k_unpack(double* __restrict__ u, const int32_t* __restrict__ idx, const double* __restrict__ buf,
                         long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) u[idx[i]] = buf[i];
}

void enqueue_pack(sc_ctx* c, const double* u, cudaStream_t st) {
  const long long n = c->xs_off.empty() ? 0 : c->xs_off.back();
  if (n) k_pack<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(u, c->d_xs_idx, c->d_xs_buf, n);
}

void enqueue_unpack(sc_ctx* c, double* u, cudaStream_t st) {
  const long long n = c->xr_off.empty() ? 0 : c->xr_off.back();
  if (n) k_unpack<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(u, c->d_xr_idx, c->d_xr_buf, n);
  SC_CUDA(cudaGetLastError());
}

// owned DOF values -> dst[canonical index] (other entries untouched); DEVICE dst
__global__ void k_scatter_owned(const double* __restrict__ u, const int32_t* __restrict__ lat,
                                const int32_t* __restrict__ dof, double* __restrict__ dst, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) dst[dof[i]] = u[lat[i]];
}

void gather_owned(sc_ctx* c, const double* d_lat, double* d_dst) {
  const long long n = (long long)c->own_dofs.size();
  if (n) k_scatter_owned<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(d_lat, c->d_own_lat, c->d_own_dof,
                                                                             d_dst, n);
  SC_CUDA(cudaGetLastError());
}

void device_upload_reference(sc_ctx* c) {
  const int n1 = c->g.p + 1;
  std::vector<double> M(SC_MAXP1 * SC_MAXP1, 0.0), K(SC_MAXP1 * SC_MAXP1, 0.0), w(SC_MAXP1, 0.0);
  for (int i = 0; i < n1; ++i) {
    w[i] = c->gll_w[i];
    for (int j = 0; j < n1; ++j) {
      M[i * n1 + j] = c->Mhat[i * n1 + j];
      K[i * n1 + j] = c->Khat[i * n1 + j];
    }
  }
  SC_CUDA(cudaMemcpyToSymbol(c_Mh, M.data(), sizeof(double) * M.size()));
  SC_CUDA(cudaMemcpyToSymbol(c_Kh, K.data(), sizeof(double) * K.size()));
  SC_CUDA(cudaMemcpyToSymbol(c_w, w.data(), sizeof(double) * w.size()));
  std::vector<double> iw(SC_MAXP1, 0.0);
  for (int i = 0; i < n1; ++i) iw[i] = 1.0 / c->gll_w[i];
  const double iw2 = 1.0 / (c->gll_w[0] + c->gll_w[c->g.p]);
  SC_CUDA(cudaMemcpyToSymbol(c_iw, iw.data(), sizeof(double) * iw.size()));
  SC_CUDA(cudaMemcpyToSymbol(c_iw2, &iw2, sizeof(double)));
  {
    // even-odd blocks of Mhat, Khat for the 3D explicit kernel (explicit3d_v2.cuh)
    std::vector<double> eo(4 * SC_EO_STRIDE);
    v2::eo_blocks(c->g.p, M.data(), K.data(), eo.data());
    SC_CUDA(cudaMemcpyToSymbol(c_EO, eo.data(), sizeof(double) * eo.size()));
  }
  SC_CUDA(cudaMalloc(&c->d_Kref, sizeof(double) * c->Kref.size()));
  SC_CUDA(cudaMemcpy(c->d_Kref, c->Kref.data(), sizeof(double) * c->Kref.size(), cudaMemcpyHostToDevice));

}

void gather_dofs(sc_ctx* c, const double* d_lat, double* d_out) {
  if (c->n_dof == 0) return;
  k_gather<<<(unsigned)((c->n_dof + 255) / 256), 256, 0, c->stream>>>(d_lat, c->d_dof_lat, d_out, c->n_dof);
  SC_CUDA(cudaGetLastError());
}

// Consistent start (reading C3): a_0 = M^-1 (f_t(0) f_x - K u_0) blockwise,
// u^d_{-1} = u^d_0 - dt v^d_0 + dt^2/2 a^d_0; v^c = v^c_0, a^c = a^c_0.
// u0, v0: DEVICE arrays of length n_dof (canonical) or nullptr.
void run_startup(sc_ctx* c, const double* u0, const double* v0) {
  const size_t latb = sizeof(double) * c->n_lat;
  c->cur = 0;
  double* A = c->d_u[0];
  double* B = c->d_u[1];
  SC_CUDA(cudaMemsetAsync(A, 0, latb, c->stream));
  SC_CUDA(cudaMemsetAsync(B, 0, latb, c->stream));
  SC_CUDA(cudaMemsetAsync(c->d_step, 0, sizeof(long long), c->stream));
  SC_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
  const unsigned gb = (unsigned)((c->n_dof + 255) / 256);
  if (u0 && c->n_dof) k_scatter<<<gb, 256, 0, c->stream>>>(u0, c->d_dof_lat, A, c->n_dof);
  double* vlat = nullptr;
  if (v0 && c->n_dof) {
    if (!c->d_vlat) SC_CUDA(cudaMalloc(&c->d_vlat, latb));
    vlat = c->d_vlat;
    SC_CUDA(cudaMemsetAsync(vlat, 0, latb, c->stream));
    k_scatter<<<gb, 256, 0, c->stream>>>(v0, c->d_dof_lat, vlat, c->n_dof);
  }
  const double dt = c->dt;
  // d part: B = u0 - dt v0 + dt^2/2 a0  (P = v0 lattice, or A with a2 = 0 when v0 == 0)
  const double* Pv = vlat ? vlat : A;
  const double a2 = vlat ? -dt : 0.0;
  launch_explicit(c, A, Pv, B, 1.0, a2, 0.5 * dt * dt, 5, c->stream);
  launch_irregular(c, A, Pv, B, 1.0, a2, 0.5 * dt * dt, c->stream);
  launch_load_d(c, B, 0.5 * dt * dt, c->stream);
  if (c->n_cl > 0 && c->integrator == 1) {
    launch_celem(c, 1, A, A, c->stream);
    k_crhs<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(c->d_b, c->d_fxc, c->d_rhs_ptr, c->d_rhs_idx,
                                                                      c->d_Y, (int)c->n_cl, c->d_ft, c->n_t,
                                                                      c->d_step, 0, nullptr);
    k_start_hrz<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(A, B, c->d_b, c->d_mc, vlat, c->d_c_lat,
                                                                           (int)c->n_cl, dt);
  } else if (c->n_cl > 0) {
    launch_celem(c, 1, A, A, c->stream);
    k_crhs<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(c->d_b, c->d_fxc, c->d_rhs_ptr, c->d_rhs_idx,
                                                                     c->d_Y, (int)c->n_cl, c->d_ft, c->n_t,
                                                                     c->d_step, 0, c->fM.d);
    launch_solve(c, c->fM, c->stream);
    if (c->integrator == 3)
      k_start_cons<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(A, B, c->d_x, c->fM.d, vlat, c->d_c_lat,
                                                                             (int)c->n_cl, dt);
    if (c->integrator == 4)   // leap-frog: u^c_0, u^c_{-1} at the fine level
      k_start_lf<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(A, c->d_vc, c->d_ac, c->d_x, c->fM.d, vlat,
                                                                           c->d_c_lat, (int)c->n_cl, dt / c->lf_m);
    else
      k_start_c<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(c->d_ac, c->d_vc, c->d_x, vlat, c->d_c_lat,
                                                                           (int)c->n_cl, c->fM.d);
  }
  SC_CUDA(cudaGetLastError());
  SC_CUDA(cudaStreamSynchronize(c->stream));
  c->host_step = 0;
  c->far_ready = false;
}

// instrumentation (sc_profile): one launch of a single sub-kernel on the context stream
void profile_launch(sc_ctx* c, int which) {
  const double* A = c->d_u[c->cur];
  double* B = c->d_u[c->cur ^ 1];
  c->far_ready = false;
  if (which == 0) launch_explicit(c, A, B, B, 2.0, -1.0, c->dt * c->dt, 5, c->stream);
  else if (which == 1) launch_celem(c, 0, A, B, c->stream);
  else if (which == 2) launch_solve(c, c->fS, c->stream);
  else launch_explicit(c, A, B, B, 2.0, -1.0, c->dt * c->dt, 4, c->stream);
}

// ---- NEXT-2: critical time step of the explicit subsystem on the device.
// Power iteration for lambda_max of M_dd^{-1} K_dd (dt_crit = 2 / omega_max): the
// operator is the explicit kernels themselves with a1 = a2 = 0, a3 = -1 and no load, applied
// to vectors that vanish off the d DOFs (so the c DOFs are held at zero: the IMEX limit is
// that of the d subsystem).  Rayleigh-type estimate (x.y)/(x.x); deterministic
// two-pass reductions.  Clobbers the state (both lattice buffers).
namespace {
__global__ void k_power_init(double* x, const uint8_t* __restrict__ nt, long long n, bool all) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t t = nt[i];
  // deterministic pseudo-random start in [0.5, 1.5) on the d DOFs
  unsigned long long z = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
  z ^= z >> 29;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 32;
  x[i] = (t == 1 || t == 2 || t == 4 || (t == 3 && all)) ? 0.5 + (double)(z >> 11) * (1.0 / 9007199254740992.0)
                                                        : 0.0;
}
// per-block partial sums of x.y, x.x, y.y
__global__ void k_dots(const double* __restrict__ x, const double* __restrict__ y, long long n, double* part) {
  __shared__ double sh[3][8];
  double a = 0.0, b = 0.0, cc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double xi = x[i], yi = y[i];
    a += xi * yi;
    b += xi * xi;
    cc += yi * yi;
  }
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    cc += __shfl_xor_sync(0xffffffffu, cc, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sh[0][w] = a;
    sh[1][w] = b;
    sh[2][w] = cc;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += sh[threadIdx.x][k];
    part[3 * blockIdx.x + threadIdx.x] = s;
  }
}
// sums the partials (fixed order), records lambda_k = (x.y)/(x.x), scale = 1/|y|
__global__ void k_dots_final(const double* part, int nblk, double* out) {
  double a = 0.0, b = 0.0, cc = 0.0;
  for (int k = 0; k < nblk; ++k) {
    a += part[3 * k];
    b += part[3 * k + 1];
    cc += part[3 * k + 2];
  }
  out[0] = a / b;
  out[1] = cc > 0.0 ? 1.0 / sqrt(cc) : 0.0;
}
__global__ void k_scale_into(double* x, const double* __restrict__ y, const double* sc, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) x[i] = y[i] * sc[1];
}
// elastic energy E = 1/2 u^T K u: the terms u_i (K u)_i summed in a
// fixed order (grid-stride per thread, warp shuffles, one partial per block, one final thread):
//   tensor-d rows  (K u)_i = M_i Y_i,  Y = M^{-1} K u from the explicit kernel,
//                  M_i = rho prod_k (h_k/2) wt(i_k)  (the lumped mass the kernel divides by)
//   irregular rows (K u)_i = Y_i / invm_i            (k_irregular with a zero load)
//   c rows         (K u)_i = -b_i                    (c-element products, k_crhs, zero load)
__global__ void k_energy_terms(const double* __restrict__ U, const double* __restrict__ Y,
                               const uint8_t* __restrict__ nt, GridP g, double mscale,
                               const int32_t* __restrict__ irr_lat, const double* __restrict__ irr_invm,
                               long long n_irr, const int32_t* __restrict__ c_lat,
                               const double* __restrict__ bc, long long n_c, long long n, double* part) {
  __shared__ double sh[32];
  double a = 0.0;
  const long long tot = n + n_irr + n_c;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    if (t < n) {
      const uint8_t ty = nt[t];
      if (ty == 1 || ty == 4) {
        long long rem = t;
        double m = mscale;
        for (int k = 0; k < g.dim; ++k) {
          const int ik = (int)(rem % g.nl[k]);
          rem /= g.nl[k];
          m *= wt(ik, g.N[k], g.p);
        }
        a += U[t] * (m * Y[t]);
      }
    } else if (t < n + n_irr) {
      const long long j = t - n;
      const int32_t L = irr_lat[j];
      a += U[L] * (Y[L] / irr_invm[j]);
    } else {
      const long long j = t - n - n_irr;
      a -= U[c_lat[j]] * bc[j];
    }
  }
  for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) b += sh[k];
    part[blockIdx.x] = b;
  }
}
__global__ void k_half_sum(const double* part, int nblk, double* out) {
  double a = 0.0;
  for (int k = 0; k < nblk; ++k) a += part[k];
  out[0] = 0.5 * a;
}
}  // namespace

// Y = A X on the explicit rows: M^{-1} K X (c^2 included) at the d DOFs; integrator 1 also the
// c rows with the HRZ mass, integrator 3 the c rows with the consistent M^cc (its factor)
static void apply_explicit_operator(sc_ctx* c, const double* X, double* Y) {
  const long long n = c->n_lat;
  SC_CUDA(cudaMemsetAsync(Y, 0, sizeof(double) * n, c->stream));
  launch_explicit(c, X, X, Y, 0.0, 0.0, -1.0, 5, c->stream);
  launch_irregular(c, X, X, Y, 0.0, 0.0, -1.0, c->stream, 0.0);
  if (c->integrator == 1 && c->n_cl > 0) {   // all DOFs explicit: the c rows with M~
    launch_celem(c, 1, X, X, c->stream);
    k_crhs<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(
        c->d_b, c->d_fxc, c->d_rhs_ptr, c->d_rhs_idx, c->d_Y, (int)c->n_cl, c->d_ft, c->n_t, c->d_step, 0, nullptr,
        0.0);
    k_hrz_apply<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(Y, c->d_b, c->d_mc, c->d_c_lat,
                                                                            (int)c->n_cl);
  } else if (c->integrator == 3 && c->n_cl > 0) {   // c rows with the consistent M^cc (its factor)
    launch_celem(c, 1, X, X, c->stream);
    k_crhs<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(
        c->d_b, c->d_fxc, c->d_rhs_ptr, c->d_rhs_idx, c->d_Y, (int)c->n_cl, c->d_ft, c->n_t, c->d_step, 0, c->fM.d,
        0.0);
    launch_solve(c, c->fM, c->stream);
    k_cons_apply<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(Y, c->d_x, c->fM.d, c->d_c_lat,
                                                                             (int)c->n_cl);
  }
}

namespace {
// diagonal mass on the lattice for the Lanczos inner product <x, y>_M = sum_i m_i x_i y_i:
// tensor-d nodes rho prod_k (h_k/2) w~(i_k) (what the explicit kernel divides by), irregular d
// nodes 1 / invm, c nodes their HRZ mass (integrator 1) or 0 (held at zero: the d subsystem)
__global__ void k_mass_lattice(double* __restrict__ dm, const uint8_t* __restrict__ nt, GridP g, double mscale,
                               long long n) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint8_t ty = nt[t];
  double m = 0.0;
  if (ty == 1 || ty == 4) {
    long long rem = t;
    m = mscale;
    for (int k = 0; k < g.dim; ++k) {
      const int ik = (int)(rem % g.nl[k]);
      rem /= g.nl[k];
      m *= wt(ik, g.N[k], g.p);
    }
  }
  dm[t] = m;
}
__global__ void k_mass_list(double* __restrict__ dm, const int32_t* __restrict__ lat, const double* __restrict__ v,
                            long long n, bool inverse) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j < n) dm[lat[j]] = inverse ? 1.0 / v[j] : v[j];
}
// per-block partial sums of sum_i m_i a_i b_i (fixed order)
__global__ void k_wdot(const double* __restrict__ a, const double* __restrict__ b, const double* __restrict__ m,
                       long long n, double* part) {
  __shared__ double sh[8];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += m[i] * a[i] * b[i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += sh[k];
    part[blockIdx.x] = t;
  }
}
// out = sum of the partials (sqrt if root)
__global__ void k_wdot_final(const double* part, int nblk, double* out, bool root) {
  double s = 0.0;
  for (int k = 0; k < nblk; ++k) s += part[k];
  *out = root ? sqrt(s) : s;
}
// Lanczos three-term step: w -= alpha v1 + beta v0 (beta = 0 at the first step)
__global__ void k_lz_orth(double* __restrict__ w, const double* __restrict__ v1, const double* __restrict__ v0,
                          const double* alpha, const double* beta, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = *alpha, b = beta ? *beta : 0.0;
  w[i] = w[i] - a * v1[i] - (beta ? b * v0[i] : 0.0);
}
__global__ void k_lz_scale(double* __restrict__ w, const double* nrm, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) w[i] = *nrm > 0.0 ? w[i] / *nrm : 0.0;
}
}  // namespace

// largest eigenvalue of the symmetric tridiagonal T (diagonal a[0..m), off-diagonal b[0..m-1))
// by bisection on Sturm sequence counts, to the last bits
static double tridiag_max_eig(const std::vector<double>& a, const std::vector<double>& b, int m) {
  double lo = a[0], hi = a[0];
  for (int i = 0; i < m; ++i) {
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  auto count_above = [&](double x) {   // eigenvalues > x = m - (eigenvalues <= x)
    int neg = 0;
    double q = 1.0;
    for (int i = 0; i < m; ++i) {
      const double bb = i > 0 ? b[i - 1] * b[i - 1] : 0.0;
      q = a[i] - x - (i > 0 ? bb / q : 0.0);
      if (q == 0.0) q = -1e-300;
      if (q < 0.0) ++neg;
    }
    return m - neg;
  };
  for (int it = 0; it < 200 && hi - lo > 4e-16 * std::fabs(hi); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (count_above(mid) > 0) lo = mid;
    else hi = mid;
  }
  return hi;
}

// Largest eigenvalue of the explicit operator.  Integrators 0 and 1: Lanczos in the M inner
// product (M diagonal, the operator M-self-adjoint), at most `iters` steps, stopped once the
// largest Ritz value changes by less than 1e-14 relative over 10 steps; integrator 3 (M^cc
// not diagonal): power iteration with the Rayleigh quotient, `iters` steps.
double estimate_lambda(sc_ctx* c, int iters) {
  const long long n = c->n_lat;
  const int nblk = 148 * 4;
  const unsigned gb = (unsigned)((n + 255) / 256);
  double* scratch = nullptr;
  SC_CUDA(cudaMalloc(&scratch, sizeof(double) * (3 * nblk + 2 * (size_t)iters + 8)));
  double* part = scratch;
  double* res = scratch + 3 * nblk;
  double* alpha = res + 2;
  double* beta = alpha + iters;
  double* X = c->d_u[0];
  double* Y = c->d_u[1];
  k_power_init<<<gb, 256, 0, c->stream>>>(X, c->d_ntype, n, c->integrator == 1 || c->integrator == 3);
  double lam = 0.0;
  if (c->integrator == 3) {
    for (int k = 0; k < iters; ++k) {
      apply_explicit_operator(c, X, Y);
      k_dots<<<nblk, 256, 0, c->stream>>>(X, Y, n, part);
      k_dots_final<<<1, 1, 0, c->stream>>>(part, nblk, res);
      k_scale_into<<<gb, 256, 0, c->stream>>>(X, Y, res, n);
    }
    double h[2] = {0.0, 0.0};
    SC_CUDA(cudaMemcpyAsync(h, res, sizeof(double) * 2, cudaMemcpyDeviceToHost, c->stream));
    SC_CUDA(cudaStreamSynchronize(c->stream));
    lam = h[0];
  } else {
    double *dm = nullptr, *W = nullptr;
    SC_CUDA(cudaMalloc(&dm, sizeof(double) * n));
    SC_CUDA(cudaMalloc(&W, sizeof(double) * n));
    double* const Wbuf = W;
    double ms = c->rho;
    for (int k = 0; k < c->g.dim; ++k) ms *= 0.5 * c->g.h[k];
    k_mass_lattice<<<gb, 256, 0, c->stream>>>(dm, c->d_ntype, c->g, ms, n);
    if (c->n_irr > 0)
      k_mass_list<<<(unsigned)((c->n_irr + 255) / 256), 256, 0, c->stream>>>(dm, c->d_irr_lat, c->d_irr_invm, c->n_irr,
                                                                               true);
    if (c->integrator == 1 && c->n_cl > 0)
      k_mass_list<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(dm, c->d_c_lat, c->d_mc, c->n_cl, false);
    // v1 = x / |x|_M
    double* V0 = Y;   // v_{j-1}
    double* V1 = X;   // v_j
    k_wdot<<<nblk, 256, 0, c->stream>>>(V1, V1, dm, n, part);
    k_wdot_final<<<1, 1, 0, c->stream>>>(part, nblk, res, true);
    k_lz_scale<<<gb, 256, 0, c->stream>>>(V1, res, n);
    std::vector<double> ha, hb;
    double prev = 0.0;
    int m = 0;
    for (int j = 0; j < iters; ++j) {
      apply_explicit_operator(c, V1, W);
      k_wdot<<<nblk, 256, 0, c->stream>>>(W, V1, dm, n, part);
      k_wdot_final<<<1, 1, 0, c->stream>>>(part, nblk, alpha + j, false);
      k_lz_orth<<<gb, 256, 0, c->stream>>>(W, V1, V0, alpha + j, j > 0 ? beta + j - 1 : nullptr, n);
      k_wdot<<<nblk, 256, 0, c->stream>>>(W, W, dm, n, part);
      k_wdot_final<<<1, 1, 0, c->stream>>>(part, nblk, beta + j, true);
      k_lz_scale<<<gb, 256, 0, c->stream>>>(W, beta + j, n);
      std::swap(V0, V1);   // v_{j-1} <- v_j
      std::swap(V1, W);    // v_j <- w / beta_j, W <- the old v_{j-1} (overwritten next step)
      m = j + 1;
      if (m % 10 == 0 || m == iters) {
        ha.resize(m);
        hb.resize(m);
        SC_CUDA(cudaMemcpyAsync(ha.data(), alpha, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
        SC_CUDA(cudaMemcpyAsync(hb.data(), beta, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
        SC_CUDA(cudaStreamSynchronize(c->stream));
        lam = tridiag_max_eig(ha, hb, m);
        if (hb[m - 1] <= 0.0 || (m >= 20 && std::fabs(lam - prev) <= 1e-14 * std::fabs(lam))) break;
        prev = lam;
      }
    }
    SC_CUDA(cudaFree(dm));
    SC_CUDA(cudaFree(Wbuf));   // W itself has rotated through the Lanczos vectors
  }
  SC_CUDA(cudaFree(scratch));
  c->far_ready = false;
  return lam;
}

// E = 1/2 u_n^T K u_n of the current state (one rank): the step kernels with zero CDM
// coefficients give M^{-1} K u on the d rows and K u on the c rows (k_energy_terms above)
double elastic_energy(sc_ctx* c) {
  const GridP& g = c->g;
  const long long n = c->n_lat;
  const double* U = c->d_u[c->cur];
  double *Y = nullptr, *bc = nullptr, *part = nullptr;
  const int nblk = 148 * 4;
  SC_CUDA(cudaMalloc(&Y, sizeof(double) * std::max<long long>(1, n)));
  SC_CUDA(cudaMalloc(&bc, sizeof(double) * std::max<long long>(1, c->n_cl)));
  SC_CUDA(cudaMalloc(&part, sizeof(double) * (nblk + 1)));
  launch_explicit(c, U, U, Y, 0.0, 0.0, -1.0, 5, c->stream);
  launch_irregular(c, U, U, Y, 0.0, 0.0, -1.0, c->stream, 0.0);
  if (c->n_cl > 0) {
    launch_celem(c, 1, U, U, c->stream);
    k_crhs<<<(unsigned)((c->n_cl + 255) / 256), 256, 0, c->stream>>>(bc, c->d_fxc, c->d_rhs_ptr, c->d_rhs_idx, c->d_Y,
                                                                       (int)c->n_cl, c->d_ft, c->n_t, c->d_step, 0,
                                                                       nullptr, 0.0);
  }
  double ms = c->rho;
  for (int k = 0; k < g.dim; ++k) ms *= 0.5 * g.h[k];
  k_energy_terms<<<nblk, 256, 0, c->stream>>>(U, Y, c->d_ntype, g, ms, c->d_irr_lat, c->d_irr_invm, c->n_irr,
                                              c->d_c_lat, bc, c->n_cl, n, part);
  k_half_sum<<<1, 1, 0, c->stream>>>(part, nblk, part + nblk);
  SC_CUDA(cudaGetLastError());
  double e = 0.0;
  SC_CUDA(cudaMemcpyAsync(&e, part + nblk, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  SC_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(Y);
  cudaFree(bc);
  cudaFree(part);
  return e;
}
