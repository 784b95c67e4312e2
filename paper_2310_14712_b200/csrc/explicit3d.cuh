// Fused explicit kernel (a1)+(a2) in 3D, register-blocked element-local sum factorisation.
//
// On the all-uncut lattice K = rho c^2 prod(h/2) sum_k (2/h_k)^2 Khat_k (x) Mhat (x) Mhat
// with ASSEMBLED 1D operators, so r' = s0 Kx My Mz u + s1 Mx Ky Mz u +
// s2 Mx My Kz u.  Each 1D operator is applied element by element ((P+1) outputs from (P+1)
// inputs held in registers: 2(P+1) FMAs per shared-memory load) and assembled at the
// element-boundary node: z by a register carry across element layers, y through a
// second shared-memory pass, x by a warp shuffle between neighbouring elements.
//
// CTA: xy tile of EX x EY elements (+1 halo element on the low side of each axis, whose
// only output is its contribution to the tile's first boundary node), streaming along z
// over EZ element layers (+1 warm-up layer that only produces the z carry).  One plane at a
// time: z-contract (registers) -> SA, SB, SU ; y pass -> BM, BT ; x pass + CDM update.
#pragma once

template <int P, int EX, int EY, int EZ, int NT>
__global__ void __launch_bounds__(NT, 2) k_explicit_3d(const double* __restrict__ U, const double* Pv, double* out,
                                                    const uint8_t* __restrict__ nt, ExpP e, int* flag) {
  constexpr int P1 = P + 1;
  constexpr int EXH = EX + 1, EYH = EY + 1;
  constexpr int RX = EXH * P + 1, RY = EYH * P + 1, TY = EY * P + 1;
  constexpr int NCOL = (RX * RY + NT - 1) / NT;
  constexpr int NYI = (RX * EYH + NT - 1) / NT;   // y-pass items per thread
  constexpr int RPW = 32 / EXH;                   // x-pass rows per warp
  extern __shared__ double smem[];
  double* SA = smem;             // [RY][RX]  Mz u   (plane)
  double* SB = SA + RY * RX;     // [RY][RX]  Kz u
  double* SU = SB + RY * RX;     // [RY][RX]  u
  double* BM = SU + RY * RX;     // [TY][RX]  My Mz u           (owned rows)
  double* BT = BM + TY * RX;     // [TY][RX]  s1 Ky Mz u + s2 My Kz u
  const int tid = threadIdx.x;
  const int Nx = e.N[0], Ny = e.N[1], Nz = e.N[2];
  const int nx = e.nl[0], ny = e.nl[1];
  const size_t pl = (size_t)nx * ny;
  const int ex0 = blockIdx.x * EX, ey0 = blockIdx.y * EY, ez0 = blockIdx.z * EZ;
  const int ex1 = min(ex0 + EX, Nx), ey1 = min(ey0 + EY, Ny), ez1 = min(ez0 + EZ, Nz);
  const int nEX = ex1 - ex0, nEY = ey1 - ey0;           // actual owned elements
  const int xr0 = (ex0 - 1) * P, yr0 = (ey0 - 1) * P;   // region origin (may be negative)
  const int gxmax = ex1 * P, gymax = ey1 * P;           // last region node (inclusive)
  const int y0 = ey0 * P;
  const int OY = nEY * P + (ey1 == Ny ? 1 : 0);         // owned rows
  const bool lastx = (ex1 == Nx);

  double u[NCOL][P1];
  double ca[NCOL], cb[NCOL];
#pragma unroll
  for (int c = 0; c < NCOL; ++c) ca[c] = cb[c] = 0.0;

  for (int ez = max(ez0 - 1, 0); ez < ez1; ++ez) {
    const bool warm = ez < ez0;
    const bool top = (ez == Nz - 1);
    // ---- load the layer's columns (P+1 planes) into registers
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const int col = tid + c * NT;
      const int ix = col % RX, iy = col / RX;
      const int gx = xr0 + ix, gy = yr0 + iy;
      const bool ok = col < RX * RY && gx >= 0 && gy >= 0 && gx <= gxmax && gy <= gymax;
      const double* base = U + gx + (size_t)nx * gy + pl * (size_t)(ez * P);
#pragma unroll
      for (int k = 0; k < P1; ++k) u[c][k] = ok ? __ldg(base + pl * k) : 0.0;
    }
    if (!warm) {
      const int np = top ? P1 : P;
      for (int k = 0; k < np; ++k) {
        // ---- z contraction for plane k -> SA, SB, SU
#pragma unroll
        for (int c = 0; c < NCOL; ++c) {
          const int col = tid + c * NT;
          if (col < RX * RY) {
            double a = 0.0, b = 0.0;
#pragma unroll
            for (int m = 0; m < P1; ++m) {
              a += c_Mh[k * P1 + m] * u[c][m];
              b += c_Kh[k * P1 + m] * u[c][m];
            }
            if (k == 0) {
              a += ca[c];
              b += cb[c];
            }
            SA[col] = a;
            SB[col] = b;
            SU[col] = u[c][k];
          }
        }
        __syncthreads();
        // ---- y pass: element-local, outputs l = 0..P-1 written, l = P added after a barrier
        double mP[NYI], tP[NYI];
#pragma unroll
        for (int q = 0; q < NYI; ++q) {
          const int it = tid + q * NT;
          const int ix = it % RX, eyl = it / RX;
          mP[q] = tP[q] = 0.0;
          if (it < RX * EYH && eyl <= nEY && (eyl > 0 || ey0 > 0)) {
            double sa[P1], sb[P1];
#pragma unroll
            for (int j = 0; j < P1; ++j) {
              sa[j] = SA[(eyl * P + j) * RX + ix];
              sb[j] = SB[(eyl * P + j) * RX + ix];
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
                mP[q] = m;
                tP[q] = t;
              }
            }
          }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NYI; ++q) {
          const int it = tid + q * NT;
          const int ix = it % RX, eyl = it / RX;
          if (it < RX * EYH && eyl <= nEY && (eyl > 0 || ey0 > 0)) {
            const int row = eyl * P;  // boundary node between element eyl and eyl+1
            if (eyl < nEY) {
              BM[row * RX + ix] += mP[q];
              BT[row * RX + ix] += tP[q];
            } else if (ey1 == Ny) {
              BM[row * RX + ix] = mP[q];
              BT[row * RX + ix] = tP[q];
            }
          }
        }
        __syncthreads();
        // ---- x pass: lane = (row, element) ; boundary nodes assembled by shfl_up
        const int warp = tid >> 5, lane = tid & 31;
        const int rin = lane / EXH, exl = lane % EXH;
        const int gz = ez * P + k;
        for (int rb = warp * RPW; rb < OY; rb += (NT / 32) * RPW) {
          const int oy = rb + rin;
          const bool act = rin < RPW && oy < OY && exl <= nEX && (exl > 0 || ex0 > 0);
          double r[P1];
#pragma unroll
          for (int l = 0; l < P1; ++l) r[l] = 0.0;
          if (act) {
            double bm[P1], bt[P1];
#pragma unroll
            for (int j = 0; j < P1; ++j) {
              bm[j] = BM[oy * RX + exl * P + j];
              bt[j] = BT[oy * RX + exl * P + j];
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
            const int gy = y0 + oy;
            const double wyz = wt(gy, Ny, P) * wt(gz, Nz, P);
            const int nl = (exl == nEX && lastx) ? P1 : P;
#pragma unroll
            for (int l = 0; l < P1; ++l) {
              if (l < nl) {
                const int gx = (ex0 - 1 + exl) * P + l;
                double rr = r[l];
                if (l == 0 && (exl > 1 || ex0 > 0)) rr += left;
                const size_t g = gx + (size_t)nx * gy + pl * gz;
                if (nt[g] == 1) {
                  const double uu = SU[(oy + P) * RX + exl * P + l];
                  const double res = e.a1 * uu + e.a2 * Pv[g] - e.coefR * rr / (wt(gx, Nx, P) * wyz);
                  out[g] = res;
                  if (!isfinite(res)) atomicExch(flag, 1);
                }
              }
            }
          }
        }
        __syncthreads();
      }
    }
    // ---- z carry: contribution of this layer to the next layer's bottom plane
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int m = 0; m < P1; ++m) {
        a += c_Mh[P * P1 + m] * u[c][m];
        b += c_Kh[P * P1 + m] * u[c][m];
      }
      ca[c] = a;
      cb[c] = b;
    }
  }
}

template <int P>
struct Tile3 {
  static constexpr int E = P <= 2 ? 8 : (P == 3 ? 7 : (P == 4 ? 5 : 4));
  static constexpr int EZ = 8;
  static constexpr int NT = 256;
  static constexpr int RX = (E + 1) * P + 1;
  static constexpr size_t smem = sizeof(double) * (3 * RX * RX + 2 * (E * P + 1) * RX);
};
