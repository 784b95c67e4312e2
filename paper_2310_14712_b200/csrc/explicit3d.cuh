// Fused explicit kernel (a1)+(a2) in 3D, register-blocked element-local sum factorisation.
//
// On the all-uncut lattice K = rho c^2 prod(h/2) sum_k (2/h_k)^2 Khat_k (x) Mhat (x) Mhat
// with ASSEMBLED 1D operators, so r' = s0 Kx My Mz u + s1 Mx Ky Mz u +
// s2 Mx My Kz u.  Each 1D operator is applied element by element ((P+1) outputs from (P+1)
// inputs held in registers) and assembled at element-boundary nodes: z by a register carry
// across element layers, y through shared memory (boundary contributions kept apart and
// added when read), x by a warp shuffle between neighbouring elements.
//
// CTA: xy tile of EX x EY elements (+1 halo element on the low side of each axis, whose
// only output is its contribution to the tile's first boundary node), streaming along z
// over EZ element layers (+1 warm-up layer that only produces the z carry).  Each layer
// ((P+1) lattice planes of the region) is staged into shared memory with cp.async
// (zero-fill outside the grid), double buffered: layer ez+1 is in flight while layer ez is
// computed.  Per plane: z-contract -> SA, SB | barrier | y pass -> BM, BT (+BMP, BTP) |
// barrier | x pass + CDM update.
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

template <int P, int EX, int EY, int EZ, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_explicit_3d(const double* __restrict__ U, const double* Pv,
                                                          double* out, const uint8_t* __restrict__ nt, ExpP e,
                                                          int* flag) {
  constexpr int P1 = P + 1;
  constexpr int EXH = EX + 1, EYH = EY + 1;
  constexpr int RX = EXH * P + 1, RY = EYH * P + 1, TY = EY * P + 1;
  constexpr int RC = RX * RY;                     // region columns
  constexpr int NCOL = (RC + NT - 1) / NT;
  constexpr int NYI = (RX * EYH + NT - 1) / NT;   // y-pass items per thread
  constexpr int RPW = 32 / EXH;                   // x-pass rows per warp
  extern __shared__ double smem[];
  double* LU = smem;                 // [2][P1][RY][RX] staged layers
  double* SA = LU + 2 * P1 * RC;     // [RY][RX]  Mz u (plane)
  double* SB = SA + RC;              // [RY][RX]  Kz u
  double* BM = SB + RC;              // [TY][RX]  My Mz u (l < P contributions)
  double* BT = BM + TY * RX;         // [TY][RX]  s1 Ky Mz u + s2 My Kz u
  double* BMP = BT + TY * RX;        // [EYH][RX] l = P contributions (boundary rows)
  double* BTP = BMP + EYH * RX;
  const int tid = threadIdx.x;
  const int Nx = e.N[0], Ny = e.N[1], Nz = e.N[2];
  const int nx = e.nl[0], ny = e.nl[1];
  const size_t pl = (size_t)nx * ny;
  const int ex0 = blockIdx.x * EX, ey0 = blockIdx.y * EY, ez0 = blockIdx.z * EZ;
  const int ex1 = min(ex0 + EX, Nx), ey1 = min(ey0 + EY, Ny), ez1 = min(ez0 + EZ, Nz);
  const int nEX = ex1 - ex0, nEY = ey1 - ey0;
  const int xr0 = (ex0 - 1) * P, yr0 = (ey0 - 1) * P;
  const int gxmax = ex1 * P, gymax = ey1 * P;
  const int y0 = ey0 * P;
  const int OY = nEY * P + (ey1 == Ny ? 1 : 0);
  const bool lastx = (ex1 == Nx);

  auto issue = [&](int ez, int buf) {
    double* dst = LU + buf * P1 * RC;
    for (int col = tid; col < RC; col += NT) {
      const int ix = col % RX, iy = col / RX;
      const int gx = xr0 + ix, gy = yr0 + iy;
      const bool ok = gx >= 0 && gy >= 0 && gx <= gxmax && gy <= gymax;
      const double* src = U + (ok ? gx + (size_t)nx * gy + pl * (size_t)(ez * P) : 0);
#pragma unroll
      for (int k = 0; k < P1; ++k) cp_async8(dst + k * RC + col, src + (ok ? pl * k : 0), ok);
    }
    cp_async_commit();
  };

  double ca[NCOL], cb[NCOL];
#pragma unroll
  for (int c = 0; c < NCOL; ++c) ca[c] = cb[c] = 0.0;
  const int ezs = max(ez0 - 1, 0);
  issue(ezs, 0);
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
    double u[NCOL][P1];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const int col = tid + c * NT;
#pragma unroll
      for (int k = 0; k < P1; ++k) u[c][k] = col < RC ? L[k * RC + col] : 0.0;
    }
    if (ez >= ez0) {
      const bool top = (ez == Nz - 1);
      const int np = top ? P1 : P;
      for (int k = 0; k < np; ++k) {
        // ---- z contraction for plane k -> SA, SB
#pragma unroll
        for (int c = 0; c < NCOL; ++c) {
          const int col = tid + c * NT;
          if (col < RC) {
            double a = k == 0 ? ca[c] : 0.0, b = k == 0 ? cb[c] : 0.0;
#pragma unroll
            for (int m = 0; m < P1; ++m) {
              a += c_Mh[k * P1 + m] * u[c][m];
              b += c_Kh[k * P1 + m] * u[c][m];
            }
            SA[col] = a;
            SB[col] = b;
          }
        }
        __syncthreads();
        // ---- y pass (element-local); l = P outputs go to BMP/BTP
#pragma unroll
        for (int q = 0; q < NYI; ++q) {
          const int it = tid + q * NT;
          const int ix = it % RX, eyl = it / RX;
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
                BMP[eyl * RX + ix] = m;
                BTP[eyl * RX + ix] = t;
              }
            }
          }
        }
        __syncthreads();
        // ---- x pass: lane = (row, element); boundary nodes assembled by shfl_up
        const int warp = tid >> 5, lane = tid & 31;
        const int rin = lane / EXH, exl = lane % EXH;
        const int gz = ez * P + k;
        const double* Lk = L + k * RC;
        for (int rb = warp * RPW; rb < OY; rb += (NT / 32) * RPW) {
          const int oy = rb + rin;
          const bool act = rin < RPW && oy < OY && exl <= nEX && (exl > 0 || ex0 > 0);
          const int q = oy / P;
          const bool brow = (oy - q * P) == 0;
          const bool hasA = oy < nEY * P;              // written by an element above (l < P)
          const bool hasP = brow && (q > 0 || ey0 > 0);  // l = P contribution of element q
          double r[P1];
#pragma unroll
          for (int l = 0; l < P1; ++l) r[l] = 0.0;
          if (act) {
            double bm[P1], bt[P1];
#pragma unroll
            for (int j = 0; j < P1; ++j) {
              const int cidx = exl * P + j;
              bm[j] = (hasA ? BM[oy * RX + cidx] : 0.0) + (hasP ? BMP[q * RX + cidx] : 0.0);
              bt[j] = (hasA ? BT[oy * RX + cidx] : 0.0) + (hasP ? BTP[q * RX + cidx] : 0.0);
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
                  const double uu = Lk[(oy + P) * RX + exl * P + l];
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
    // ---- z carry for the next layer's bottom plane
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
    __syncthreads();  // all reads of this layer's buffer done before it is refilled
  }
}

template <int P>
struct Tile3 {
  static constexpr int E = P <= 2 ? 8 : (P == 3 ? 7 : (P == 4 ? 5 : 3));
  static constexpr int EZ = 8;
  static constexpr int NT = 256;
  static constexpr int MINB = P <= 4 ? 3 : 1;
  static constexpr int RX = (E + 1) * P + 1;
  static constexpr int TY = E * P + 1;
  static constexpr size_t smem = sizeof(double) * (2 * (P + 1) * RX * RX + 2 * RX * RX + 2 * TY * RX + 2 * (E + 1) * RX);
};
