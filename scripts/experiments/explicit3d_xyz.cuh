// Fused explicit kernel (a1)+(a2) in 3D: separated x, y, z passes.
//
// On the all-uncut lattice K = rho c^2 prod(h/2) sum_k (2/h_k)^2 Khat_k (x) Mhat (x) Mhat with
// ASSEMBLED 1D operators, so with s_k = (2/h_k)^2
//   r' = s1 [ Mz S + sig2 Kz T ],   S = sig0 My P1 + Ky P2,   T = My P2,   P1 = Kx u,  P2 = Mx u,
// sig0 = s0/s1, sig2 = s2/s1 (the three 1D operators of each axis commute with the others).
// The passes run in that order on a CTA tile of EX x EY elements streaming along z:
//  * the tile's region (one halo element on the low x / y side) of each element layer's P new
//    lattice planes is staged into shared memory by the TMA engine: a 1D tensor map over the
//    whole lattice array (its rows, N*P+1 doubles, are not 16-byte aligned, so a 3D map is not
//    possible), one box per (plane, row), completing on an mbarrier, double buffered;
//  * X pass: one lane per (plane, row, x element), the element's P+1 nodes contracted with
//    Khat and Mhat in even-odd form, the element-boundary node assembled with a warp shuffle;
//    it runs on the tile's output columns for every region row (rows of the y halo included);
//  * Y pass: one thread per (plane, output column, y element), even-odd, the element's top
//    node contribution kept apart (added by the Z pass);
//  * Z pass: one thread per output (x, y) column, the element layer's P+1 planes contracted
//    with Mhat and Khat (even-odd) and the layer's bottom plane assembled with a register
//    carry from the layer below; fused with the CDM update of the column's nodes
//    u_{n+1} = a1 u_n + a2 u_{n-1} - coefR s1 r / (w_x w_y w_z).
// Compared with the element-local kernel (explicit3d.cuh) no halo element is contracted in
// z and y, and no node is contracted twice in z: 30% fewer FP64 operations per node.
#pragma once
// EXPERIMENT (not built into libsc): separated x, y, z passes; measured slower
// (profiles/r2_variants.txt).
#include <cuda.h>

#include "../../paper_2310_14712_b200/csrc/explicit3d_v2.cuh"   // even-odd helpers (v2::eo_*) and c_EO

namespace xyz {

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
  }
}
// one 1D TMA box (the map's box size) from element index x of the flat lattice array
__device__ __forceinline__ void tma_row(void* dst, const CUtensorMap* map, long long x, uint64_t* bar) {
  // 1D tensor coordinates are 32-bit: the lattice of config 5 has 2.6e8 < 2^31 nodes
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"((int)x), "r"(su32(bar))
      : "memory");
}

template <int P, int EX, int EY>
struct Geo {
  static constexpr int P1 = P + 1, EXH = EX + 1, EYH = EY + 1;
  static constexpr int RX = EXH * P + 1;        // region columns (low halo element + top node)
  // staged row: the TMA box starts at the even element at or below the row's first node (box
  // starts must be 16-byte aligned in global memory) and lands 128-byte aligned in shared memory
  static constexpr int RXS = (RX + 1 + 15) / 16 * 16;
  static constexpr int RY = EYH * P + 1;        // region rows
  static constexpr int OXS = EX * P + 1;        // output columns (last one: the grid's high face)
  static constexpr int TYS = EY * P + 1;        // output rows
  static constexpr int STG = ((P * RY * RXS + 15) / 16) * 16;   // one stage buffer (doubles, 128 B multiple)
  static constexpr int PB = P * RY * OXS;       // P1 or P2
  static constexpr int SB = P * TYS * OXS;      // S or T
  static constexpr int HB = P * EYH * OXS;      // SP or TP (y elements' top-node contributions)
  static constexpr size_t smem = sizeof(double) * (2 * STG + 2 * PB + 2 * SB + 2 * HB) + 64;
};

template <int P, int EX, int EY, int NT, bool INT, bool CLEAN>
__device__ __forceinline__ void tile(const CUtensorMap* map, const double* __restrict__ U, const double* Pv,
                                     double* out, const uint8_t* __restrict__ nt, const ExpP& e, int* flag,
                                     const int3 tb, unsigned& use) {
  using G = Geo<P, EX, EY>;
  constexpr int P1 = P + 1, NE = v2::EOdims<P>::NE, NO = v2::EOdims<P>::NO;
  constexpr int EXH = G::EXH, EYH = G::EYH, RXS = G::RXS, RY = G::RY, OXS = G::OXS, TYS = G::TYS;
  constexpr int NW = NT / 32;
  constexpr int GX = 32 / EXH;                                 // X-pass rows per warp
  constexpr int NXR = (P * RY + NW * GX - 1) / (NW * GX);      // X-pass rounds
  constexpr int NYR = (P * EYH * OXS + NT - 1) / NT;           // Y-pass rounds
  constexpr int NZI = ((OXS - 1) * (TYS - 1) + NT - 1) / NT;   // Z-pass columns per thread (interior)
  constexpr int NZM = (OXS * TYS + NT - 1) / NT;               // ... (boundary tiles)
  constexpr int NZ = INT ? NZI : NZM;
  const double* EM = c_EO;
  const double* OM = c_EO + SC_EO_STRIDE;
  const double* EK = c_EO + 2 * SC_EO_STRIDE;
  const double* OK = c_EO + 3 * SC_EO_STRIDE;
  extern __shared__ __align__(128) double xsm[];
  double* stage = xsm;                  // [2][P][RY][RXS]
  double* B1 = stage + 2 * G::STG;       // P1 [P][RY][OXS]
  double* B2 = B1 + G::PB;               // P2
  double* BS = B2 + G::PB;               // S  [P][TYS][OXS]
  double* BT = BS + G::SB;               // T
  double* HS = BT + G::SB;               // SP [P][EYH][OXS]
  double* HT = HS + G::HB;               // TP
  uint64_t* bar = reinterpret_cast<uint64_t*>(HT + G::HB);   // [2]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Nx = e.N[0], Ny = e.N[1], Nz = e.N[2];
  const int nx = e.nl[0], ny = e.nl[1];
  const long long pl = (long long)nx * ny;
  const int ex0 = tb.x * EX, ey0 = tb.y * EY, ez0 = tb.z * e.ezl;
  const int ex1 = INT ? ex0 + EX : min(ex0 + EX, Nx), ey1 = INT ? ey0 + EY : min(ey0 + EY, Ny);
  const int ez1 = min(ez0 + e.ezl, Nz);
  const int nEX = INT ? EX : ex1 - ex0, nEY = INT ? EY : ey1 - ey0;
  const bool lastx = INT ? false : ex1 == Nx, lasty = INT ? false : ey1 == Ny;
  const int xr0 = (ex0 - 1) * P, yr0 = (ey0 - 1) * P;   // region origin (may be -P)
  const int OXA = INT ? EX * P : nEX * P + (lastx ? 1 : 0);   // owned columns
  const int OYA = INT ? EY * P : nEY * P + (lasty ? 1 : 0);   // owned rows
  const double sig0 = e.s[0] / e.s[1], sig2 = e.s[2] / e.s[1];
  const int ylo_r = INT ? 0 : max(0, -yr0), yhi_r = INT ? RY : min(RY, ny - yr0);   // rows inside the lattice
  const int first = ez0 > 0 ? ez0 - 1 : 0;   // first element layer streamed (a warm-up one if ez0 > 0)
  // lattice offset of the region's (0, 0) node in plane L*P + 1 + k: rbase + pl * (L*P + 1 + k)
  const long long rbase = (long long)xr0 + (long long)nx * yr0;

  // ---- TMA producer (warp 0): plane slots [k0, k0 + npl) of layer L's stage <- lattice planes
  // L*P + 1 + k (the base step loads only lattice plane first*P into slot P-1); each row's box
  // starts at the even element at or below it (16-byte aligned global start)
  auto produce = [&](int L, int k0, int npl, int buf) {
    if (warp != 0) return;
    double* dst = stage + buf * G::STG;
    const int nyr = yhi_r - ylo_r;
    if (lane == 0) mbar_expect(&bar[buf], (unsigned)(npl * nyr * RXS * 8));
    __syncwarp();
    for (int i = lane; i < npl * nyr; i += 32) {
      const int kk = i / nyr, iy = ylo_r + (i - kk * nyr), k = k0 + kk;
      const long long g = rbase + (long long)nx * iy + pl * ((long long)L * P + 1 + k);
      tma_row(dst + (k * RY + iy) * RXS, map, g & ~1LL, &bar[buf]);
    }
  };

  // ---- X-pass items (regular layers): lane group xg of a warp takes region row r of round t
  const int xg = lane / EXH, exl = lane - xg * EXH;   // lane group (row) and x element (0 = halo)
  const bool xel = INT || (ex0 - 1 + exl >= 0 && ex0 - 1 + exl < Nx);   // element inside the grid
  const bool xwr = exl > 0 && (INT || exl <= nEX);                        // writes output columns
  const bool lastel = exl == (INT ? EX : nEX);   // the tile's last element: writes its top node too

  // one X item: element exl of stage row `so` (shifted by sh), valid v; writes at `d` (>= 0)
  auto xitem = [&](const double* st, int so, int d, bool v) {
    double u[P1];
#pragma unroll
    for (int j = 0; j < P1; ++j) u[j] = v ? st[so + j] : 0.0;
    double eu[NE], ou[NO], p1[P1], p2[P1];
    v2::eo_split<P>(u, eu, ou);
    v2::eo_apply<P>(EK, OK, eu, ou, p1);
    v2::eo_apply<P>(EM, OM, eu, ou, p2);
    const double l1 = __shfl_up_sync(0xffffffffu, p1[P], 1);
    const double l2 = __shfl_up_sync(0xffffffffu, p2[P], 1);
    if (d >= 0) {
      double* d1 = B1 + d;
      double* d2 = B2 + d;
      d1[0] = p1[0] + l1;
      d2[0] = p2[0] + l2;
#pragma unroll
      for (int j = 1; j < P; ++j) {
        d1[j] = p1[j];
        d2[j] = p2[j];
      }
      if (lastel) {   // partial unless the grid ends there
        d1[P] = p1[P];
        d2[P] = p2[P];
      }
    }
  };

  // ---- Y-pass items: it = tid + t NT -> (column ox, y element eyl, plane slot k)
  auto yitem = [&](int so, int d, int h, bool v) {
    double a[P1], b[P1];
#pragma unroll
    for (int j = 0; j < P1; ++j) {
      a[j] = v ? B1[so + j * OXS] : 0.0;
      b[j] = v ? B2[so + j * OXS] : 0.0;
    }
    double ea[NE], oa[NO], eb[NE], ob[NO], sv[P1], tv[P1];
    v2::eo_split<P>(a, ea, oa);
    v2::eo_split<P>(b, eb, ob);
    v2::eo_apply2<P>(EK, OK, eb, ob, EM, OM, ea, oa, sig0, sv);
    v2::eo_apply<P>(EM, OM, eb, ob, tv);
    if (d >= 0) {
#pragma unroll
      for (int j = 0; j < P; ++j) {
        BS[d + j * OXS] = sv[j];
        BT[d + j * OXS] = tv[j];
      }
    }
    HS[h] = sv[P];
    HT[h] = tv[P];
  };

  // ---- Z-pass columns: the tile's owned (x, y) columns, it = tid + q NT
  int zo[NZ];          // lattice offset of the column in plane 0 (x + nx y), -1: none
  int zs[NZ];          // S/T offset; < 0: no S entry (the top boundary row)
  int zh[NZ];          // SP/TP offset for a vertex row, -1 otherwise
  double zc[NZ];       // coefR s1 / (w_x w_y)
#pragma unroll
  for (int q = 0; q < NZ; ++q) {
    const int it = tid + q * NT;
    const int oy = it / OXA, ox = it - oy * OXA;
    const bool own = oy < OYA;
    const int gx = ex0 * P + ox, gy = ey0 * P + oy;
    zo[q] = own ? gx + nx * gy : -1;
    zs[q] = oy < nEY * P ? oy * OXS + ox : -1;
    const int ly = oy % P, lx = ox % P;
    zh[q] = ly == 0 ? (oy / P) * OXS + ox : -1;
    const double iwx = lx ? c_iw[lx] : ((gx / P > 0 && gx / P < Nx) ? c_iw2 : c_iw[0]);
    const double iwy = ly ? c_iw[ly] : ((gy / P > 0 && gy / P < Ny) ? c_iw2 : c_iw[0]);
    zc[q] = e.coefR * e.s[1] * iwx * iwy;
  }
  auto zread = [&](int q, int k, double& s, double& t) {
    s = zs[q] >= 0 ? BS[k * (TYS * OXS) + zs[q]] : 0.0;
    t = zs[q] >= 0 ? BT[k * (TYS * OXS) + zs[q]] : 0.0;
    if (zh[q] >= 0) {
      s += HS[k * (EYH * OXS) + zh[q]];
      t += HT[k * (EYH * OXS) + zh[q]];
    }
  };
  double S0[NZ], T0[NZ], car[NZ];

  if (use == 0 && tid == 0) {
    mbar_init(&bar[0]);
    mbar_init(&bar[1]);
  }
  __syncthreads();
  const unsigned u0 = use;
  produce(first - 1, P - 1, 1, u0 & 1);   // the base plane first*P, slot P-1
  produce(first, 0, P, (u0 + 1) & 1);
#pragma unroll
  for (int q = 0; q < NZ; ++q) car[q] = 0.0;
  bool bad = false;
  for (int L = first - 1; L < ez1; ++L) {
    const unsigned cu = use++;
    const int buf = cu & 1;
    const bool base = L == first - 1;
    mbar_wait(&bar[buf], (cu >> 1) & 1);
    const double* st = stage + buf * G::STG;
    if (base) {
      for (int rb = warp * GX; rb < RY; rb += NW * GX) {
        const int iy = rb + xg;
        const bool ok = xg < GX && iy < RY;
        bool valid = ok && xel;
        if constexpr (!INT) valid = valid && iy >= ylo_r && iy < yhi_r;
        const long long g0 = rbase + (long long)nx * iy + pl * ((long long)L * P + P);
        const int row = (P - 1) * RY + iy;
        xitem(st, row * RXS + exl * P + (int)(g0 & 1), (ok && xwr) ? row * OXS + (exl - 1) * P : -1, valid);
      }
    } else {
#pragma unroll
      for (int t = 0; t < NXR; ++t) {
        const int rb = warp * GX + t * NW * GX;
        if (rb < P * RY) {   // warp-uniform
          const int r = rb + xg;
          const bool ok = xg < GX && r < P * RY;
          const int k = r / RY, iy = r - k * RY;
          bool valid = ok && xel;
          if constexpr (!INT) valid = valid && iy >= ylo_r && iy < yhi_r;
          const long long g0 = rbase + (long long)nx * iy + pl * ((long long)L * P + 1 + k);
          const int row = k * RY + iy;
          xitem(st, row * RXS + exl * P + (int)(g0 & 1), (ok && xwr) ? row * OXS + (exl - 1) * P : -1, valid);
        }
      }
    }
    __syncthreads();
    if (L + 2 < ez1) produce(L + 2, 0, P, buf);
    if (base) {
      for (int it = tid; it < EYH * OXS; it += NT) {
        const int ox = it % OXS, eyl = it / OXS, k = P - 1;
        const bool yin = INT || (ey0 - 1 + eyl >= 0 && ey0 - 1 + eyl < Ny);
        yitem((k * RY + eyl * P) * OXS + ox, eyl > 0 ? (k * TYS + (eyl - 1) * P) * OXS + ox : -1,
              (k * EYH + eyl) * OXS + ox, yin);
      }
    } else {
#pragma unroll
      for (int t = 0; t < NYR; ++t) {
        const int it = tid + t * NT;
        if (it < P * EYH * OXS) {
          const int ox = it % OXS, rest = it / OXS;
          const int eyl = rest % EYH, k = rest / EYH;
          const bool yin = INT || (ey0 - 1 + eyl >= 0 && ey0 - 1 + eyl < Ny);
          yitem((k * RY + eyl * P) * OXS + ox, eyl > 0 ? (k * TYS + (eyl - 1) * P) * OXS + ox : -1,
                (k * EYH + eyl) * OXS + ox, yin);
        }
      }
    }
    __syncthreads();
    // ---- Z pass (+ CDM update of this layer's planes)
    const bool upd = L >= ez0, top = L == Nz - 1;
#pragma unroll
    for (int q = 0; q < NZ; ++q) {
      if (zo[q] < 0) continue;
      if (base) {
        zread(q, P - 1, S0[q], T0[q]);
        continue;
      }
      const long long g0 = zo[q] + pl * ((long long)L * P);
      double s[P1], t[P1];
      s[0] = S0[q];
      t[0] = T0[q];
#pragma unroll
      for (int k = 1; k < P1; ++k) zread(q, k - 1, s[k], t[k]);
      double es[NE], os[NO], et[NE], ot[NO], r[P1];
      v2::eo_split<P>(s, es, os);
      v2::eo_split<P>(t, et, ot);
      v2::eo_apply2<P>(EM, OM, es, os, EK, OK, et, ot, sig2, r);
      r[0] += car[q];
      car[q] = r[P];
      S0[q] = s[P];
      T0[q] = t[P];
      if (upd) {
#pragma unroll
        for (int l = 0; l < P1; ++l) {
          if (l == P && !top) break;
          const long long g = g0 + pl * l;
          bool w = true;
          if constexpr (!CLEAN) w = (e.want >> __ldg(nt + g)) & 1;
          if (w) {
            const double iwz = (l > 0 && l < P) ? c_iw[l] : (l == P ? c_iw[0] : (L > 0 ? c_iw2 : c_iw[0]));
            const double res = fma(e.a1, U[g], fma(e.a2, Pv[g], -(zc[q] * iwz) * r[l]));
            out[g] = res;
            bad |= !isfinite(res);
          }
        }
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

template <int P, int EX, int EY, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_xyz(const __grid_constant__ CUtensorMap map, const double* __restrict__ U,
                                                  const double* Pv, double* out, const uint8_t* __restrict__ nt,
                                                  ExpP e, int* flag) {
  unsigned use = 0;   // stage-buffer uses so far (mbarrier phase parities)
  for (int tt = blockIdx.x; tt < e.ntiles; tt += gridDim.x) {
    const int id = e.tiles ? e.tiles[tt] : tt;
    const int3 tb = tile_of(e, tt);
    const bool clean = e.clean && e.clean[id];
    const bool in = tb.x > 0 && tb.y > 0 && (tb.x + 1) * EX < e.N[0] && (tb.y + 1) * EY < e.N[1];
    if (in) {
      if (clean) tile<P, EX, EY, NT, true, true>(&map, U, Pv, out, nt, e, flag, tb, use);
      else tile<P, EX, EY, NT, true, false>(&map, U, Pv, out, nt, e, flag, tb, use);
    } else {
      if (clean) tile<P, EX, EY, NT, false, true>(&map, U, Pv, out, nt, e, flag, tb, use);
      else tile<P, EX, EY, NT, false, false>(&map, U, Pv, out, nt, e, flag, tb, use);
    }
  }
}

}  // namespace xyz
