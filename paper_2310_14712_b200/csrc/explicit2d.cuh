// Fused explicit kernel (a1)+(a2) in 2D: r' = s0 Kx My u + s1 Mx Ky u on the all-uncut
// lattice (assembled 1D operators), register-blocked element-local
// contractions as in explicit3d.cuh: the tile (EX x EY elements + 1 low-side halo element
// per axis) is staged in shared memory; y pass element-local (boundary rows assembled after
// a barrier); x pass with lanes = (row, element) and boundary nodes assembled by shfl_up.
#pragma once

template <int P, int EX, int EY, int NT>
__device__ __forceinline__ void explicit2d_tile(const double* __restrict__ U, const double* Pv, double* out,
                                                const uint8_t* __restrict__ nt, const ExpP& e, int* flag,
                                                const int3 tb) {
  constexpr int P1 = P + 1;
  constexpr int EXH = EX + 1, EYH = EY + 1;
  constexpr int RX = EXH * P + 1, RY = EYH * P + 1, TY = EY * P + 1;
  constexpr int NYI = (RX * EYH + NT - 1) / NT;
  constexpr int RPW = 32 / EXH;
  __shared__ double SU[RY * RX];
  __shared__ double BM[TY * RX];
  __shared__ double BK[TY * RX];
  const int tid = threadIdx.x;
  const int Nx = e.N[0], Ny = e.N[1];
  const int nx = e.nl[0];
  const int ex0 = tb.x * EX, ey0 = tb.y * EY;
  const int ex1 = min(ex0 + EX, Nx), ey1 = min(ey0 + EY, Ny);
  const int nEX = ex1 - ex0, nEY = ey1 - ey0;
  const int xr0 = (ex0 - 1) * P, yr0 = (ey0 - 1) * P;
  const int gxmax = ex1 * P, gymax = ey1 * P;
  const int y0 = ey0 * P;
  const int OY = nEY * P + (ey1 == Ny ? 1 : 0);
  const bool lastx = (ex1 == Nx);
  for (int col = tid; col < RX * RY; col += NT) {
    const int ix = col % RX, iy = col / RX;
    const int gx = xr0 + ix, gy = yr0 + iy;
    const bool ok = gx >= 0 && gy >= 0 && gx <= gxmax && gy <= gymax;
    SU[col] = ok ? __ldg(U + gx + (size_t)nx * gy) : 0.0;
  }
  __syncthreads();
  double mP[NYI], kP[NYI];
#pragma unroll
  for (int q = 0; q < NYI; ++q) {
    const int it = tid + q * NT;
    const int ix = it % RX, eyl = it / RX;
    mP[q] = kP[q] = 0.0;
    if (it < RX * EYH && eyl <= nEY && (eyl > 0 || ey0 > 0)) {
      double su[P1];
#pragma unroll
      for (int j = 0; j < P1; ++j) su[j] = SU[(eyl * P + j) * RX + ix];
#pragma unroll
      for (int l = 0; l < P1; ++l) {
        double m = 0.0, k = 0.0;
#pragma unroll
        for (int j = 0; j < P1; ++j) {
          m += c_Mh[l * P1 + j] * su[j];
          k += c_Kh[l * P1 + j] * su[j];
        }
        if (l < P) {
          if (eyl > 0) {
            BM[((eyl - 1) * P + l) * RX + ix] = m;
            BK[((eyl - 1) * P + l) * RX + ix] = k;
          }
        } else {
          mP[q] = m;
          kP[q] = k;
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
      const int row = eyl * P;
      if (eyl < nEY) {
        BM[row * RX + ix] += mP[q];
        BK[row * RX + ix] += kP[q];
      } else if (ey1 == Ny) {
        BM[row * RX + ix] = mP[q];
        BK[row * RX + ix] = kP[q];
      }
    }
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int rin = lane / EXH, exl = lane % EXH;
  for (int rb = warp * RPW; rb < OY; rb += (NT / 32) * RPW) {
    const int oy = rb + rin;
    const bool act = rin < RPW && oy < OY && exl <= nEX && (exl > 0 || ex0 > 0);
    double r[P1];
#pragma unroll
    for (int l = 0; l < P1; ++l) r[l] = 0.0;
    if (act) {
      double bm[P1], bk[P1];
#pragma unroll
      for (int j = 0; j < P1; ++j) {
        bm[j] = BM[oy * RX + exl * P + j];
        bk[j] = BK[oy * RX + exl * P + j];
      }
#pragma unroll
      for (int l = 0; l < P1; ++l) {
        double kx = 0.0, mx = 0.0;
#pragma unroll
        for (int j = 0; j < P1; ++j) {
          kx += c_Kh[l * P1 + j] * bm[j];
          mx += c_Mh[l * P1 + j] * bk[j];
        }
        r[l] = e.s[0] * kx + e.s[1] * mx;
      }
    }
    const double left = __shfl_up_sync(0xffffffffu, r[P], 1);
    if (act && exl > 0) {
      const int gy = y0 + oy;
      const double cy = e.coefR * inv_wt(gy, Ny, P);
      const int nl = (exl == nEX && lastx) ? P1 : P;
#pragma unroll
      for (int l = 0; l < P1; ++l) {
        if (l < nl) {
          const int gx = (ex0 - 1 + exl) * P + l;
          double rr = r[l];
          if (l == 0 && (exl > 1 || ex0 > 0)) rr += left;
          const size_t g = gx + (size_t)nx * gy;
          if ((e.want >> nt[g]) & 1) {
            const double uu = SU[(oy + P) * RX + exl * P + l];
            const double res = e.a1 * uu + e.a2 * Pv[g] - cy * inv_wt(gx, Nx, P) * rr;
            out[g] = res;
            if (!isfinite(res)) atomicExch(flag, 1);
          }
        }
      }
    }
  }
}

template <int P, int EX, int EY, int NT>
__global__ void __launch_bounds__(NT) k_explicit_2d(const double* __restrict__ U, const double* Pv, double* out,
                                                    const uint8_t* __restrict__ nt, ExpP e, int* flag) {
  for (int tt = blockIdx.x; tt < e.ntiles; tt += gridDim.x) {
    explicit2d_tile<P, EX, EY, NT>(U, Pv, out, nt, e, flag, tile_of(e, tt));
    __syncthreads();   // shared tile buffers reused by the next tile
  }
}

template <int P>
struct Tile2v {
  static constexpr int E = P <= 2 ? 10 : (P <= 4 ? 8 : (P <= 6 ? 5 : 4));
  static constexpr int NT = 256;
};
