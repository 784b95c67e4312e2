// Fused explicit kernel (a1)+(a2) in 3D, register-blocked element-local sum factorisation.
//
// On the all-uncut lattice K = rho c^2 prod(h/2) sum_k (2/h_k)^2 Khat_k (x) Mhat (x) Mhat
// with ASSEMBLED 1D operators, so r' = s0 Kx My Mz u + s1 Mx Ky Mz u +
// s2 Mx My Kz u.  Each 1D operator is applied element by element ((P+1) outputs from (P+1)
// inputs held in registers) and assembled at element-boundary nodes: z by a register carry
// across element layers, y through shared memory (boundary contributions kept apart and
// added when read), x by a warp shuffle between neighbouring x elements.
//
// CTA: xy tile of EX x EY elements (+1 halo element on the low side of each axis, whose
// only output is its contribution to the tile's first boundary node), streaming along z
// over EZ element layers (+1 warm-up layer that only produces the z carry).
//  * each layer ((P+1) lattice planes of the region) is staged into shared memory with
//    cp.async (zero fill outside the grid), double buffered (layer ez+1 in flight while
//    layer ez is computed);
//  * z and y contractions are thread-local: a "column item" (x, y-element) holds its
//    (P+1) x (P+1) block of u in registers and produces the y-element's outputs for every
//    plane; results go to BM/BT (double-buffered per plane parity);
//  * one barrier per plane, then the x pass: a "row item" (row, x-element) contracts in x,
//    assembles the shared node with shfl_up and applies the CDM update; u_{n-1} and the node
//    type of the NEXT plane are prefetched into registers;
//  * the lumped-mass division uses precomputed reciprocal GLL weights.
#pragma once

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// reciprocal of the assembled 1D GLL weight of lattice node i
__device__ __forceinline__ double inv_wt(int i, int e_cnt, int P) {
  const int l = i % P, e = i / P;
  if (l) return c_iw[l];
  return (e > 0 && e < e_cnt) ? c_iw2 : c_iw[0];
}

template <int P, int EX, int EY, int NT, bool SPV, bool INT>
__device__ __forceinline__ void explicit3d_tile(const double* __restrict__ U, const double* Pv, double* out,
                                                const uint8_t* __restrict__ nt, const ExpP& e, int* flag,
                                                const int3 tb, const bool clean) {
  constexpr int P1 = P + 1;
  constexpr int EXH = EX + 1, EYH = EY + 1;
  constexpr int RX = EXH * P + 1, RY = EYH * P + 1, TY = EY * P + 1;
  constexpr int RC = RX * RY;                     // region columns
  constexpr int NYI = (RX * EYH + NT - 1) / NT;   // column items per thread
  constexpr int RPW = 32 / EXH;                   // x-pass rows per warp
  constexpr int NW = NT / 32;
  constexpr int NXI = (TY + NW * RPW - 1) / (NW * RPW);   // row-item rounds per warp
  extern __shared__ double smem[];
  double* LU = smem;                   // [2][P1][RY][RX] staged layers
  double* BMb = LU + 2 * P1 * RC;      // [2][TY][RX]  My Mz u (l < P contributions)
  double* BTb = BMb + 2 * TY * RX;     // [2][TY][RX]  s1 Ky Mz u + s2 My Kz u
  double* BMPb = BTb + 2 * TY * RX;    // [2][EYH][RX] l = P contributions (boundary rows)
  double* BTPb = BMPb + 2 * EYH * RX;
  constexpr int OXP = EX * P + 1;      // output columns of the tile
  double* SPb = BTPb + 2 * EYH * RX;   // SPV: [2][P1][TY][OXP] staged u_{n-1} of the layer's outputs
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int Nx = e.N[0], Ny = e.N[1], Nz = e.N[2];
  const int nx = e.nl[0], ny = e.nl[1];
  const size_t pl = (size_t)nx * ny;
  const int EZ = e.ezl;   // element layers per tile along z (runtime, step.cu)
  const int ex0 = tb.x * EX, ey0 = tb.y * EY, ez0 = tb.z * EZ;
  // INT: an interior tile (full EX x EY elements, neither on a low nor on a high x/y face of
  // the box): every boundary test below folds at compile time
  const int ex1 = INT ? ex0 + EX : min(ex0 + EX, Nx), ey1 = INT ? ey0 + EY : min(ey0 + EY, Ny);
  const int ez1 = min(ez0 + EZ, Nz);
  const int nEX = INT ? EX : ex1 - ex0, nEY = INT ? EY : ey1 - ey0;
  const bool xlo = INT || ex0 > 0, ylo = INT || ey0 > 0;   // a halo element exists below
  const int xr0 = (ex0 - 1) * P, yr0 = (ey0 - 1) * P;
  const int gxmax = ex1 * P, gymax = ey1 * P;
  const int y0 = ey0 * P;
  const int OY = INT ? EY * P : nEY * P + (ey1 == Ny ? 1 : 0);
  const bool lastx = INT ? false : (ex1 == Nx);
  const int rin = lane / EXH, exl = lane % EXH;

  auto issue = [&](int ez, int buf) {
    double* dst = LU + buf * P1 * RC;
    for (int col = tid; col < RC; col += NT) {
      const int ix = col % RX, iy = col / RX;
      const int gx = xr0 + ix, gy = yr0 + iy;
      const bool ok = INT || (gx >= 0 && gy >= 0 && gx <= gxmax && gy <= gymax);
      const double* src = U + (ok ? gx + (size_t)nx * gy + pl * (size_t)(ez * P) : 0);
#pragma unroll
      for (int k = 0; k < P1; ++k) cp_async8(dst + k * RC + col, src + (ok ? pl * k : 0), ok);
    }
    if constexpr (SPV) {
      // u_{n-1} at the layer's output nodes (the x pass reads it from shared memory)
      if (ez >= ez0) {
        double* sp = SPb + buf * P1 * TY * OXP;
        const int OXW = nEX * P + (lastx ? 1 : 0);
        const int npl = (ez == Nz - 1) ? P1 : P;
        // warp per output row (no integer division), lanes along x
        const double* pv0 = Pv + (size_t)(ex0 * P) + (size_t)nx * y0 + pl * (size_t)(ez * P);
        for (int k = 0; k < npl; ++k)
          for (int oy = warp; oy < OY; oy += NW)
            if (lane < OXW)
              cp_async8(sp + (k * TY + oy) * OXP + lane, pv0 + (size_t)nx * oy + pl * (size_t)k + lane, true);
      }
    }
    cp_async_commit();
  };

  // row-item prefetch of u_{n-1} and node types for one plane
  double pv[NXI][P1];
  uint8_t ntv[NXI][P1];
  auto prefetch = [&](int gz) {
#pragma unroll
    for (int q = 0; q < NXI; ++q) {
      const int oy = (warp + q * NW) * RPW + rin;
      const bool act = rin < RPW && oy < OY && exl > 0 && exl <= nEX;
      const int gy = y0 + oy;
#pragma unroll
      for (int l = 0; l < P1; ++l) {
        const int gx = (ex0 - 1 + exl) * P + l;
        const bool ok = act && (l < P || (exl == nEX && lastx)) && gz < e.nl[2];
        const size_t g = gx + (size_t)nx * gy + pl * gz;
        // clean tile: every node it owns is tensor-d of a wanted type (setup_step_structures)
        ntv[q][l] = ok ? (clean ? (uint8_t)1 : __ldg(nt + g)) : (uint8_t)0;
        if constexpr (!SPV) pv[q][l] = ok ? Pv[g] : 0.0;
      }
    }
  };

  bool bad = false;                  // a non-finite update (reported once per tile)
  double ca[NYI][P1], cb[NYI][P1];   // z carries of the column items' P+1 rows
#pragma unroll
  for (int q = 0; q < NYI; ++q)
#pragma unroll
    for (int j = 0; j < P1; ++j) ca[q][j] = cb[q][j] = 0.0;
  const int ezs = max(ez0 - 1, 0);
  issue(ezs, 0);
  int pp = 0;  // plane parity (BM/BT double buffer)
  prefetch(ez0 * P);
  for (int ez = ezs; ez < ez1; ++ez) {
    const int buf = (ez - ezs) & 1;
    if (ez + 1 < ez1) {
      issue(ez + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* L = LU + buf * P1 * RC;
    const bool warm = ez < ez0;
    const bool top = (ez == Nz - 1);
    const int np = warm ? 0 : (top ? P1 : P);
    // column items: (x, y-element) blocks of u in registers: u[q][row j][plane m]
    double u[NYI][P1][P1];
#pragma unroll
    for (int q = 0; q < NYI; ++q) {
      const int it = tid + q * NT;
      const int ix = it % RX, eyl = it / RX;
      const bool ok = it < RX * EYH;
#pragma unroll
      for (int j = 0; j < P1; ++j)
#pragma unroll
        for (int m = 0; m < P1; ++m) u[q][j][m] = ok ? L[m * RC + (eyl * P + j) * RX + ix] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < P1; ++k) {
      if (k >= np) break;
      double* BM = BMb + pp * TY * RX;
      double* BT = BTb + pp * TY * RX;
      double* BMP = BMPb + pp * EYH * RX;
      double* BTP = BTPb + pp * EYH * RX;
      // ---- z then y contraction (thread-local)
#pragma unroll
      for (int q = 0; q < NYI; ++q) {
        const int it = tid + q * NT;
        const int ix = it % RX, eyl = it / RX;
        if (it < RX * EYH && eyl <= nEY && (eyl > 0 || ylo)) {
          double sa[P1], sb[P1];
#pragma unroll
          for (int j = 0; j < P1; ++j) {
            double a = k == 0 ? ca[q][j] : 0.0, b = k == 0 ? cb[q][j] : 0.0;
#pragma unroll
            for (int m = 0; m < P1; ++m) {
              a += c_Mh[k * P1 + m] * u[q][j][m];
              b += c_Kh[k * P1 + m] * u[q][j][m];
            }
            sa[j] = a;
            sb[j] = b;
          }
#pragma unroll
          for (int l = 0; l < P1; ++l) {
            double m = 0.0, tk = 0.0, tm = 0.0;
#pragma unroll
            for (int j = 0; j < P1; ++j) {
              m += c_Mh[l * P1 + j] * sa[j];
              tk += c_Kh[l * P1 + j] * sa[j];
              tm += c_Mh[l * P1 + j] * sb[j];
            }
            const double t = e.s[1] * tk + e.s[2] * tm;
            if (l < P) {
              if (eyl > 0) {
                BM[((eyl - 1) * P + l) * RX + ix] = m;
                BT[((eyl - 1) * P + l) * RX + ix] = t;
              }
            } else {
              BMP[eyl * RX + ix] = m;
              BTP[eyl * RX + ix] = t;
            }
          }
        }
      }
      __syncthreads();
      // ---- x pass + CDM update
      const int gz = ez * P + k;
      const double* Lk = L + k * RC;
      double pvc[NXI][P1];
      uint8_t ntc[NXI][P1];
#pragma unroll
      for (int q = 0; q < NXI; ++q)
#pragma unroll
        for (int l = 0; l < P1; ++l) {
          if constexpr (!SPV) pvc[q][l] = pv[q][l];
          ntc[q][l] = ntv[q][l];
        }
      prefetch(k + 1 < np ? gz + 1 : (ez + 1) * P);   // next plane (next layer's plane 0)
      const double iwz = inv_wt(gz, Nz, P);
#pragma unroll
      for (int q = 0; q < NXI; ++q) {
        const int oy = (warp + q * NW) * RPW + rin;
        const bool act = rin < RPW && oy < OY && exl <= nEX && (exl > 0 || xlo);
        const int qq = oy / P;
        const bool hasA = oy < nEY * P;
        const bool hasP = (oy - qq * P) == 0 && (qq > 0 || ylo);
        double r[P1];
#pragma unroll
        for (int l = 0; l < P1; ++l) r[l] = 0.0;
        if (act) {
          double bm[P1], bt[P1];
#pragma unroll
          for (int j = 0; j < P1; ++j) {
            const int cidx = exl * P + j;
            bm[j] = (hasA ? BM[oy * RX + cidx] : 0.0) + (hasP ? BMP[qq * RX + cidx] : 0.0);
            bt[j] = (hasA ? BT[oy * RX + cidx] : 0.0) + (hasP ? BTP[qq * RX + cidx] : 0.0);
          }
#pragma unroll
          for (int l = 0; l < P1; ++l) {
            double kx = 0.0, mx = 0.0;
#pragma unroll
            for (int j = 0; j < P1; ++j) {
              kx += c_Kh[l * P1 + j] * bm[j];
              mx += c_Mh[l * P1 + j] * bt[j];
            }
            r[l] = e.s[0] * kx + mx;
          }
        }
        const double left = __shfl_up_sync(0xffffffffu, r[P], 1);
        if (act && exl > 0) {
          // per row item: pointers and the lumped-mass reciprocals hoisted out of the node loop
          const int gy = y0 + oy;
          const int xe = ex0 - 1 + exl;                 // x element of this row item
          const double cyz = e.coefR * inv_wt(gy, Ny, P) * iwz;
          double* orow = out + (size_t)nx * gy + pl * gz + (size_t)xe * P;
          const double* urow = Lk + (oy + P) * RX + exl * P;
          const double* prow = SPV ? SPb + ((buf * P1 + k) * TY + oy) * OXP + (exl - 1) * P : nullptr;
          const double iw0 = (xe > 0) ? c_iw2 : c_iw[0];           // node xe*P (left boundary)
          const double iwP = (xe + 1 < Nx) ? c_iw2 : c_iw[0];      // node (xe+1)*P
#pragma unroll
          for (int l = 0; l < P1; ++l) {
            if ((e.want >> ntc[q][l]) & 1) {
              double rr = r[l];
              if (l == 0 && (exl > 1 || xlo)) rr += left;
              double pvv;
              if constexpr (SPV) pvv = prow[l];
              else pvv = pvc[q][l];
              const double iwx = l == 0 ? iw0 : (l == P ? iwP : c_iw[l]);
              const double res = e.a1 * urow[l] + e.a2 * pvv - cyz * iwx * rr;
              orow[l] = res;
              bad |= !isfinite(res);
            }
          }
        }
      }
      pp ^= 1;
    }
    // ---- z carries for the next layer's bottom plane
#pragma unroll
    for (int q = 0; q < NYI; ++q)
#pragma unroll
      for (int j = 0; j < P1; ++j) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int m = 0; m < P1; ++m) {
          a += c_Mh[P * P1 + m] * u[q][j][m];
          b += c_Kh[P * P1 + m] * u[q][j][m];
        }
        ca[q][j] = a;
        cb[q][j] = b;
      }
    __syncthreads();  // all reads of this layer's buffer done before it is refilled
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

// grid-stride loop over the tiles (a capped grid leaves SM resources to a concurrent kernel)
template <int P, int EX, int EY, int NT, int MINB, bool SPV>
__global__ void __launch_bounds__(NT, MINB) k_explicit_3d(const double* __restrict__ U, const double* Pv,
                                                          double* out, const uint8_t* __restrict__ nt, ExpP e,
                                                          int* flag) {
  for (int tt = blockIdx.x; tt < e.ntiles; tt += gridDim.x) {
    const int id = e.tiles ? e.tiles[tt] : tt;
    const int3 tb = tile_of(e, tt);
    const bool clean = e.clean && e.clean[id];
    if (tb.x > 0 && tb.y > 0 && (tb.x + 1) * EX < e.N[0] && (tb.y + 1) * EY < e.N[1])
      explicit3d_tile<P, EX, EY, NT, SPV, true>(U, Pv, out, nt, e, flag, tb, clean);
    else
      explicit3d_tile<P, EX, EY, NT, SPV, false>(U, Pv, out, nt, e, flag, tb, clean);
  }
}

// Tile shapes (EX = E along x, EY along y): the z+y phase has RX*(EY+1) column items and the
// x phase (EY*P+1) rows of (E+1) lanes; NT is sized so both keep most threads busy (one item
// each).  p = 4 (config 5; harness scripts/exp_harness.cu, profiles/r2_variants.txt): E = 8,
// EY = 4, NT = 192, 2 CTAs/SM at ~160 registers without spills 2.66 ms; 6x5 2.74, 7x4 2.76, 9x3
// 2.79; every 224-thread shape (capped at 128 registers: 6x6 3.12, 9x4 3.01, 12x3 3.10) and the
// 3-CTA shapes (8x3 at 160 threads 2.94) are slower.
#ifndef EXP4_E
#define EXP4_E 8
#endif
#ifndef EXP4_EY
#define EXP4_EY 4
#endif
#ifndef EXP4_NT
#define EXP4_NT 192
#endif
#ifndef EXP4_MINB
#define EXP4_MINB 2
#endif
#ifndef EXP4_SPV
#define EXP4_SPV 0
#endif
template <int P>
struct Tile3 {
  static constexpr int E = P <= 2 ? 8 : (P == 3 ? 7 : (P == 4 ? EXP4_E : 3));
  // p = 3 (config 4, harness at 64^3): 7x6 elements at 192 threads 0.123 ms vs 7x7 at 224 0.138
  static constexpr int EY = P == 4 ? EXP4_EY : (P == 3 ? 6 : E);
  static constexpr int EZ = 8;    // default element layers per tile (+1 warm-up layer)
  static constexpr int NT = P == 3 ? 192 : (P == 4 ? EXP4_NT : 256);
  static constexpr int MINB = P == 3 ? 2 : (P == 4 ? EXP4_MINB : (P <= 2 ? 2 : 1));
  static constexpr bool SPV = P == 3 || (P == 4 && EXP4_SPV);   // u_{n-1} staged through shared memory
  static constexpr int RX = (E + 1) * P + 1;
  static constexpr int RY = (EY + 1) * P + 1;
  static constexpr int TY = EY * P + 1;
  static constexpr size_t smem = sizeof(double) * (2 * (P + 1) * RX * RY + 4 * TY * RX + 4 * (EY + 1) * RX +
                                                   (SPV ? 2 * (P + 1) * TY * (E * P + 1) : 0));
};
