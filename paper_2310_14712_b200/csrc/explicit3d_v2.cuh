// Fused explicit kernel (a1)+(a2) in 3D, instruction-lean rewrite of explicit3d.cuh.
//
// Same data flow as explicit3d.cuh: K = rho c^2 prod(h/2) sum_k (2/h_k)^2 x
// Khat_k (x) Mhat (x) Mhat with ASSEMBLED 1D operators, so
//   r' = s1 [ sig0 Kx My Mz u + Mx (Ky Mz u + sig2 My Kz u) ],  sig0 = s0/s1, sig2 = s2/s1,
// each 1D operator applied element by element and assembled at element-boundary nodes (z by
// a register carry across element layers, y through shared memory, x by a warp shuffle).
// What changed against the r1 kernel (its ncu source capture, profiles/r2_explicit_v2.txt:
// 34% of the issued instructions were DFMA, the rest constant reloads, address arithmetic,
// register zeroing and indexed constant loads):
//  * even-odd (persymmetric) form of Mhat, Khat on the GLL nodes for the y and x operators:
//    v -> (v_j + v_{P-j}, v_j - v_{P-j}) halves the matrix products (c_EO, host-computed);
//  * no zero-initialised accumulators (chains start with a multiply), no indexed constant
//    loads (GLL reciprocal weights selected by compile-time local indices), per-tile hoisted
//    addressing, compile-time tile geometry for interior tiles;
//  * clean tiles (every owned node a wanted tensor-d node) skip the node-type loads.
#pragma once

namespace v2 {

// even-odd blocks of Mhat and Khat: NE x NE even, NO x NO odd parts
//   E[i][j] = (A[i][j] + A[i][P-j]) / 2 (j < NO), E[i][mid] = A[i][mid] (i < NO),
//   E[mid][j] = A[mid][j], O[i][j] = (A[i][j] - A[i][P-j]) / 2
// with y_i = (E e)_i + (O o)_i, y_{P-i} = (E e)_i - (O o)_i, y_mid = (E e)_mid for
// e_j = v_j + v_{P-j}, o_j = v_j - v_{P-j}, e_mid = v_mid.
template <int P>
struct EOdims {
  static constexpr int P1 = P + 1, NO = P1 / 2, NE = P1 - NO;
};

template <int P>
__device__ __forceinline__ void eo_split(const double (&v)[P + 1], double (&e)[EOdims<P>::NE],
                                         double (&o)[EOdims<P>::NO]) {
  constexpr int NO = EOdims<P>::NO;
#pragma unroll
  for (int j = 0; j < NO; ++j) {
    e[j] = v[j] + v[P - j];
    o[j] = v[j] - v[P - j];
  }
  if constexpr (EOdims<P>::NE > NO) e[NO] = v[NO];
}

// y = A v from the split (e, o); which: 0 Mhat, 1 Khat
template <int P>
__device__ __forceinline__ void eo_apply(const double* __restrict__ E, const double* __restrict__ O,
                                         const double (&e)[EOdims<P>::NE], const double (&o)[EOdims<P>::NO],
                                         double (&y)[P + 1]) {
  constexpr int NE = EOdims<P>::NE, NO = EOdims<P>::NO;
  double ye[NE], yo[NO];
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    double s = E[i * NE] * e[0];
#pragma unroll
    for (int j = 1; j < NE; ++j) s = fma(E[i * NE + j], e[j], s);
    ye[i] = s;
  }
#pragma unroll
  for (int i = 0; i < NO; ++i) {
    double s = O[i * NO] * o[0];
#pragma unroll
    for (int j = 1; j < NO; ++j) s = fma(O[i * NO + j], o[j], s);
    yo[i] = s;
  }
#pragma unroll
  for (int i = 0; i < NO; ++i) {
    y[i] = ye[i] + yo[i];
    y[P - i] = ye[i] - yo[i];
  }
  if constexpr (NE > NO) y[NO] = ye[NO];
}

// y = A1 v1 + sig * A2 v2 (two operators on two inputs, one merge)
template <int P>
__device__ __forceinline__ void eo_apply2(const double* __restrict__ E1, const double* __restrict__ O1,
                                          const double (&e1)[EOdims<P>::NE], const double (&o1)[EOdims<P>::NO],
                                          const double* __restrict__ E2, const double* __restrict__ O2,
                                          const double (&e2)[EOdims<P>::NE], const double (&o2)[EOdims<P>::NO],
                                          double sig, double (&y)[P + 1]) {
  constexpr int NE = EOdims<P>::NE, NO = EOdims<P>::NO;
  double ye[NE], yo[NO];
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    double t = E2[i * NE] * e2[0];
#pragma unroll
    for (int j = 1; j < NE; ++j) t = fma(E2[i * NE + j], e2[j], t);
    double s = sig * t;
#pragma unroll
    for (int j = 0; j < NE; ++j) s = fma(E1[i * NE + j], e1[j], s);
    ye[i] = s;
  }
#pragma unroll
  for (int i = 0; i < NO; ++i) {
    double t = O2[i * NO] * o2[0];
#pragma unroll
    for (int j = 1; j < NO; ++j) t = fma(O2[i * NO + j], o2[j], t);
    double s = sig * t;
#pragma unroll
    for (int j = 0; j < NO; ++j) s = fma(O1[i * NO + j], o1[j], s);
    yo[i] = s;
  }
#pragma unroll
  for (int i = 0; i < NO; ++i) {
    y[i] = ye[i] + yo[i];
    y[P - i] = ye[i] - yo[i];
  }
  if constexpr (NE > NO) y[NO] = ye[NO];
}

}  // namespace v2

// even-odd blocks in constant memory: [EM | OM | EK | OK], each padded to (SC_MAXP1/2+1)^2
#define SC_EO_STRIDE ((SC_MAXP1 / 2 + 1) * (SC_MAXP1 / 2 + 1))
__constant__ double c_EO[4 * SC_EO_STRIDE];

namespace v2 {

// host: even-odd blocks from Mhat, Khat ((P+1)^2 row-major)
inline void eo_blocks(int P, const double* M, const double* K, double* out /* 4*SC_EO_STRIDE */) {
  const int P1 = P + 1, NO = P1 / 2, NE = P1 - NO;
  for (int i = 0; i < 4 * SC_EO_STRIDE; ++i) out[i] = 0.0;
  const double* A[2] = {M, K};
  for (int w = 0; w < 2; ++w) {
    double* E = out + (2 * w) * SC_EO_STRIDE;
    double* O = out + (2 * w + 1) * SC_EO_STRIDE;
    const double* a = A[w];
    for (int i = 0; i < NE; ++i)
      for (int j = 0; j < NE; ++j) {
        double v;
        if (i < NO) v = j < NO ? 0.5 * (a[i * P1 + j] + a[i * P1 + (P - j)]) : a[i * P1 + j];
        else v = a[i * P1 + j];   // middle row (P even)
        E[i * NE + j] = v;
      }
    for (int i = 0; i < NO; ++i)
      for (int j = 0; j < NO; ++j) O[i * NO + j] = 0.5 * (a[i * P1 + j] - a[i * P1 + (P - j)]);
  }
}

template <int P, int EX, int EY, int NT, bool INT, bool CLEAN>
__device__ __forceinline__ void tile3(const double* __restrict__ U, const double* Pv, double* out,
                                      const uint8_t* __restrict__ nt,
                                      const ExpP& e, int* flag, const int3 tb) {
  constexpr int P1 = P + 1, NE = EOdims<P>::NE, NO = EOdims<P>::NO;
  constexpr int EXH = EX + 1, EYH = EY + 1;
  constexpr int RX = EXH * P + 1, RY = EYH * P + 1, TY = EY * P + 1;
  constexpr int RXP = RX + (RX & 1);              // padded row (16-byte aligned pairs)
  constexpr int RC = RXP * RY;                    // staged layer plane
  constexpr int NYI = (RX * EYH + NT - 1) / NT;   // column items per thread
  constexpr int RPW = 32 / EXH;                   // x-pass rows per warp
  constexpr int NW = NT / 32;
  constexpr int NXS = (EY + 1 + RPW - 1) / RPW * RPW + EY * (P - 1);   // x-pass row slots (row_of)
  constexpr int NXI = (NXS + NW * RPW - 1) / (NW * RPW);
  const double* EM = c_EO;
  const double* OM = c_EO + SC_EO_STRIDE;
  const double* EK = c_EO + 2 * SC_EO_STRIDE;
  const double* OK = c_EO + 3 * SC_EO_STRIDE;
  extern __shared__ double smem[];
  double* LU = smem;                    // [2][P1][RY][RXP]
  double* BMb = LU + 2 * P1 * RC;       // [2][TY][RXP]   My Mz u (l < P contributions)
  double* BTb = BMb + 2 * TY * RXP;     // [2][TY][RXP]   Ky Mz u + sig2 My Kz u
  double* BMPb = BTb + 2 * TY * RXP;    // [2][EYH][RXP]  l = P contributions (boundary rows)
  double* BTPb = BMPb + 2 * EYH * RXP;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int Nx = e.N[0], Ny = e.N[1], Nz = e.N[2];
  const int nx = e.nl[0], ny = e.nl[1];
  const size_t pl = (size_t)nx * ny;
  const int EZ = e.ezl;
  const int ex0 = tb.x * EX, ey0 = tb.y * EY, ez0 = tb.z * EZ;
  const int ex1 = INT ? ex0 + EX : min(ex0 + EX, Nx), ey1 = INT ? ey0 + EY : min(ey0 + EY, Ny);
  const int ez1 = min(ez0 + EZ, Nz);
  const int nEX = INT ? EX : ex1 - ex0, nEY = INT ? EY : ey1 - ey0;
  const bool xlo = INT || ex0 > 0, ylo = INT || ey0 > 0;
  const int xr0 = (ex0 - 1) * P, yr0 = (ey0 - 1) * P;
  const int gxmax = ex1 * P, gymax = ey1 * P;
  const int y0 = ey0 * P;
  const int OY = INT ? EY * P : nEY * P + (ey1 == Ny ? 1 : 0);
  const bool lastx = INT ? false : (ex1 == Nx);
  const int rin = lane / EXH, exl = lane - (lane / EXH) * EXH;
  const double sig0 = e.s[0] / e.s[1], sig2 = e.s[2] / e.s[1];

  // stage layer ez: warp per region row, lanes along x (no index division)
  auto issue = [&](int ez, int buf) {
    double* dst = LU + buf * P1 * RC;
    const double* base = U + (size_t)(ez * P) * pl + xr0;
    for (int iy = warp; iy < RY; iy += NW) {
      const int gy = yr0 + iy;
      const bool oky = INT || (gy >= 0 && gy <= gymax);
      for (int ix = lane; ix < RX; ix += 32) {
        const int gx = xr0 + ix;
        const bool ok = oky && (INT || (gx >= 0 && gx <= gxmax));
        const double* src = ok ? base + ix + (size_t)nx * gy : U;
        double* d = dst + iy * RXP + ix;
#pragma unroll
        for (int k = 0; k < P1; ++k) cp_async8(d + k * RC, src + (ok ? pl * k : 0), ok);
      }
    }
    cp_async_commit();
  };

  // x-pass row of slot (warp, round q, lane group rin): the element-boundary ("vertex") rows
  // first, padded to whole warps, then the interior rows, so that the vertex rows' extra
  // BMP/BTP reads are warp-uniform; -1: no row
  auto row_of = [&](int q) {
    constexpr int NV = EY + 1, NVP = (NV + RPW - 1) / RPW * RPW, NI = EY * (P - 1);
    const int sl = (warp + q * NW) * RPW + rin;
    if (rin >= RPW) return -1;
    if (sl < NV) return sl * P;
    if (sl < NVP || P == 1) return -1;
    const int t = sl - NVP;
    if (t >= NI) return -1;
    return (t / (P - 1)) * P + 1 + t % (P - 1);
  };

  // ---- per-thread constants of the x-pass row items (hoisted out of the plane loop)
  int xoff[NXI];          // offset of the item's first output node in a lattice plane
  int sof[NXI];           // offset of the item's element in the BM/BT rows
  int sofP[NXI];          // offset in the BMP/BTP rows (vertex rows), -1 if none
  double cy[NXI];         // coefR * iwy
  bool act[NXI], hasA[NXI];
#pragma unroll
  for (int q = 0; q < NXI; ++q) {
    const int oyr = row_of(q);
    const int oy = oyr < 0 ? 0 : oyr;
    act[q] = oyr >= 0 && oy < OY && exl <= nEX && (exl > 0 || xlo);
    const int qq = oy / P, ly = oy - qq * P;
    hasA[q] = oy < nEY * P;
    const bool hasP = ly == 0 && (qq > 0 || ylo);
    sof[q] = oy * RXP + exl * P;
    sofP[q] = hasP ? qq * RXP + exl * P : -1;
    const int gy = y0 + oy;
    const int ey = gy / P;
    const double iwy = ly ? c_iw[ly] : ((ey > 0 && ey < Ny) ? c_iw2 : c_iw[0]);
    cy[q] = e.coefR * e.s[1] * iwy;
    xoff[q] = (ex0 - 1 + exl) * P + nx * gy;
  }
  const int xe = ex0 - 1 + exl;
  const double iw0 = (xe > 0) ? c_iw2 : c_iw[0];
  const double iwP = (xe + 1 < Nx) ? c_iw2 : c_iw[0];

  // ---- column items (x, y-element) of the z+y phase
  int coff[NYI], boff[NYI], bpoff[NYI];
  bool cok[NYI];
#pragma unroll
  for (int q = 0; q < NYI; ++q) {
    const int it = tid + q * NT;
    const int eyl = it / RX, ix = it - eyl * RX;
    cok[q] = it < RX * EYH && eyl <= nEY && (eyl > 0 || ylo);
    coff[q] = (eyl * P) * RXP + ix;
    boff[q] = eyl > 0 ? ((eyl - 1) * P) * RXP + ix : -1;
    bpoff[q] = eyl * RXP + ix;
  }

  bool bad = false;
  double ca[NYI][P1], cb[NYI][P1];   // z carries of the column items' P+1 rows (0 below the grid)
#pragma unroll
  for (int q = 0; q < NYI; ++q)
#pragma unroll
    for (int j = 0; j < P1; ++j) ca[q][j] = cb[q][j] = 0.0;
  const int ezs = max(ez0 - 1, 0);
  issue(ezs, 0);
  int pp = 0;
  // u_{n-1} of the next plane (row items), prefetched one plane ahead
  double pv[NXI][P1];
  uint8_t ntv[NXI][P1];
  auto prefetch = [&](int gz) {
#pragma unroll
    for (int q = 0; q < NXI; ++q) {
      const size_t g = (size_t)xoff[q] + pl * gz;
      const bool ok = act[q] && exl > 0 && gz < e.nl[2];
#pragma unroll
      for (int l = 0; l < P1; ++l) {
        const bool okl = ok && (l < P || (exl == nEX && lastx));
        pv[q][l] = okl ? Pv[g + l] : 0.0;
        if constexpr (!CLEAN) ntv[q][l] = okl ? __ldg(nt + g + l) : (uint8_t)0;
      }
    }
  };
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
    double u[NYI][P1][P1];   // u[q][row j][plane m]
#pragma unroll
    for (int q = 0; q < NYI; ++q)
#pragma unroll
      for (int j = 0; j < P1; ++j)
#pragma unroll
        for (int m = 0; m < P1; ++m) u[q][j][m] = cok[q] ? L[m * RC + coff[q] + j * RXP] : 0.0;
    if (!warm) {
#pragma unroll
      for (int k = 0; k < P1; ++k) {
        if (k == P && !top) break;
        double* BM = BMb + pp * TY * RXP;
        double* BT = BTb + pp * TY * RXP;
        double* BMP = BMPb + pp * EYH * RXP;
        double* BTP = BTPb + pp * EYH * RXP;
        // ---- z (plane k of the layer, element-local + carry) then y (even-odd)
#pragma unroll
        for (int q = 0; q < NYI; ++q) {
          if (cok[q]) {
            double a[P1], b[P1];
#pragma unroll
            for (int j = 0; j < P1; ++j) {
              double s = c_Mh[k * P1] * u[q][j][0], t = c_Kh[k * P1] * u[q][j][0];
              if (k == 0) {
                s = fma(c_Mh[0], u[q][j][0], ca[q][j]);
                t = fma(c_Kh[0], u[q][j][0], cb[q][j]);
              }
#pragma unroll
              for (int m = 1; m < P1; ++m) {
                s = fma(c_Mh[k * P1 + m], u[q][j][m], s);
                t = fma(c_Kh[k * P1 + m], u[q][j][m], t);
              }
              a[j] = s;
              b[j] = t;
            }
            double ea[NE], oa[NO], eb[NE], ob[NO];
            eo_split<P>(a, ea, oa);
            eo_split<P>(b, eb, ob);
            double cm[P1], ct[P1];
            eo_apply<P>(EM, OM, ea, oa, cm);
            eo_apply2<P>(EK, OK, ea, oa, EM, OM, eb, ob, sig2, ct);
            if (boff[q] >= 0) {
#pragma unroll
              for (int l = 0; l < P; ++l) {
                BM[boff[q] + l * RXP] = cm[l];
                BT[boff[q] + l * RXP] = ct[l];
              }
            }
            BMP[bpoff[q]] = cm[P];
            BTP[bpoff[q]] = ct[P];
          }
        }
        __syncthreads();
        // ---- x pass (even-odd) + CDM update of plane k
        const int gz = ez * P + k;
        const double* Lk = L + k * RC;
        // lumped-mass reciprocal of plane k: interior planes compile-time, the layer's bottom
        // plane an element boundary unless on the grid's bottom face, plane P only on the top face
        const double iwzt = (k > 0 && k < P) ? c_iw[k] : (k == P ? c_iw[0] : ((ez > 0) ? c_iw2 : c_iw[0]));
#pragma unroll
        for (int q = 0; q < NXI; ++q) {
          double r[P1];
          if (act[q]) {
            double bm[P1], bt[P1];
#pragma unroll
            for (int j = 0; j < P1; ++j) {
              bm[j] = hasA[q] ? BM[sof[q] + j] : 0.0;
              bt[j] = hasA[q] ? BT[sof[q] + j] : 0.0;
            }
            if (sofP[q] >= 0) {
#pragma unroll
              for (int j = 0; j < P1; ++j) {
                bm[j] += BMP[sofP[q] + j];
                bt[j] += BTP[sofP[q] + j];
              }
            }
            double em[NE], om[NO], et[NE], ot[NO];
            eo_split<P>(bm, em, om);
            eo_split<P>(bt, et, ot);
            eo_apply2<P>(EM, OM, et, ot, EK, OK, em, om, sig0, r);
          } else {
#pragma unroll
            for (int l = 0; l < P1; ++l) r[l] = 0.0;
          }
          const double left = __shfl_up_sync(0xffffffffu, r[P], 1);
          if (act[q] && exl > 0) {
            const double cyz = cy[q] * iwzt;
            double* orow = out + (size_t)xoff[q] + pl * gz;
            const double* urow = Lk + sof[q] + RXP * P;   // u_n at the item's nodes (row oy + P)
            if (xlo || exl > 1) r[0] += left;
#pragma unroll
            for (int l = 0; l < P1; ++l) {
              if (l == P && !(exl == nEX && lastx)) break;
              bool w = true;
              if constexpr (!CLEAN) w = (e.want >> ntv[q][l]) & 1;
              if (w) {
                const double iwx = l == 0 ? iw0 : (l == P ? iwP : c_iw[l]);
                const double res = fma(e.a1, urow[l], fma(e.a2, pv[q][l], -(cyz * iwx) * r[l]));
                orow[l] = res;
                bad |= !isfinite(res);
              }
            }
          }
        }
        // u_{n-1} of the next plane (the next layer's plane 0 after k = P - 1), in flight
        // during the next plane's z+y phase
        prefetch(gz + 1);
        pp ^= 1;
      }
    }
    // ---- z carries for the next layer's bottom plane
#pragma unroll
    for (int q = 0; q < NYI; ++q)
#pragma unroll
      for (int j = 0; j < P1; ++j) {
        double a = c_Mh[P * P1] * u[q][j][0], b = c_Kh[P * P1] * u[q][j][0];
#pragma unroll
        for (int m = 1; m < P1; ++m) {
          a = fma(c_Mh[P * P1 + m], u[q][j][m], a);
          b = fma(c_Kh[P * P1 + m], u[q][j][m], b);
        }
        ca[q][j] = a;
        cb[q][j] = b;
      }
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

template <int P, int EX, int EY, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_exp3(const double* __restrict__ U, const double* Pv, double* out,
                                                   const uint8_t* __restrict__ nt, ExpP e, int* flag) {
  for (int tt = blockIdx.x; tt < e.ntiles; tt += gridDim.x) {
    const int id = e.tiles ? e.tiles[tt] : tt;
    const int3 tb = tile_of(e, tt);
    const bool clean = e.clean && e.clean[id];
    const bool in = tb.x > 0 && tb.y > 0 && (tb.x + 1) * EX < e.N[0] && (tb.y + 1) * EY < e.N[1];
    if (in) {
      if (clean) tile3<P, EX, EY, NT, true, true>(U, Pv, out, nt, e, flag, tb);
      else tile3<P, EX, EY, NT, true, false>(U, Pv, out, nt, e, flag, tb);
    } else {
      if (clean) tile3<P, EX, EY, NT, false, true>(U, Pv, out, nt, e, flag, tb);
      else tile3<P, EX, EY, NT, false, false>(U, Pv, out, nt, e, flag, tb);
    }
  }
}

template <int P, int EX, int EY>
constexpr size_t smem3() {
  constexpr int EXH = EX + 1, EYH = EY + 1;
  constexpr int RX = EXH * P + 1, RY = EYH * P + 1, TY = EY * P + 1;
  constexpr int RXP = RX + (RX & 1);
  return sizeof(double) * (2 * (P + 1) * RXP * RY + 4 * TY * RXP + 4 * EYH * RXP);
}

}  // namespace v2
