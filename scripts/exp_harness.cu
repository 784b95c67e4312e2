// Kernel experiments for the 3D explicit step (a1)+(a2), outside the library: a synthetic
// all-uncut lattice (random u_n, u_{n-1}), the product kernel (explicit3d.cuh) against a
// candidate, element-wise comparison and CUDA-event timing.  Diagnostics only (not product).
// The r1 kernel (explicit3d.cuh) is the baseline; the candidate is chosen at compile time:
//   -DWITH_V2 (the product kernel, explicit3d_v2.cuh), -DWITH_V2 -DWITH_V2T (its TMA-staged
//   variant, scripts/experiments/), -DWITH_XYZ (separated passes, scripts/experiments/):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -DWITH_V2 -o scripts/exp_harness_v2 scripts/exp_harness.cu
//   scripts/exp_harness N [reps] [mask]   (N^3 elements of order 4; mask: random unwanted nodes)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2310_14712_b200/csrc/explicit_common.cuh"
#include "../paper_2310_14712_b200/csrc/explicit3d.cuh"
#ifdef WITH_V2
#ifdef WITH_V2T
#include "experiments/explicit3d_v2_tma.cuh"
#else
#include "../paper_2310_14712_b200/csrc/explicit3d_v2.cuh"
#endif
#ifndef V2_EX
#define V2_EX 6
#endif
#ifndef V2_EY
#define V2_EY 6
#endif
#ifndef V2_NT
#define V2_NT 224
#endif
#ifndef V2_MINB
#define V2_MINB 2
#endif
#ifndef V2_EZL
#define V2_EZL 16
#endif
namespace v2 {
template <int P>
void launch(const double* U, double* out, const uint8_t* nt, ExpP e, int* flag, cudaStream_t st, bool first) {
  constexpr size_t sm = smem3<P, V2_EX, V2_EY>();
  auto k = k_exp3<P, V2_EX, V2_EY, V2_NT, V2_MINB>;
  if (first) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) exit(3);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    printf("v2 <%d,%d,%d,%d,%d>: %d regs, %zu B smem, %d B local\n", P, V2_EX, V2_EY, V2_NT, V2_MINB, fa.numRegs, sm,
           (int)fa.localSizeBytes);
  }
  e.ezl = V2_EZL;
  e.tg[0] = (e.N[0] + V2_EX - 1) / V2_EX;
  e.tg[1] = (e.N[1] + V2_EY - 1) / V2_EY;
  e.ntiles = e.tg[0] * e.tg[1] * ((e.N[2] + e.ezl - 1) / e.ezl);
  k<<<e.ntiles, V2_NT, sm, st>>>(U, out, out, nt, e, flag);
}
}  // namespace v2
#endif

#ifdef WITH_XYZ
#include "experiments/explicit3d_xyz.cuh"
#ifndef XYZ_EX
#define XYZ_EX 6
#endif
#ifndef XYZ_EY
#define XYZ_EY 4
#endif
#ifndef XYZ_NT
#define XYZ_NT 256
#endif
#ifndef XYZ_MINB
#define XYZ_MINB 2
#endif
#ifndef XYZ_EZL
#define XYZ_EZL 16
#endif
#include <cudaTypedefs.h>
namespace xyz {
template <int P>
void launch(const double* U, double* out, const uint8_t* nt, ExpP e, int* flag, cudaStream_t st, bool first) {
  using G = Geo<P, XYZ_EX, XYZ_EY>;
  auto k = k_xyz<P, XYZ_EX, XYZ_EY, XYZ_NT, XYZ_MINB>;
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess || !enc) {
      printf("no cuTensorMapEncodeTiled\n");
      exit(4);
    }
  }
  CUtensorMap map;
  const cuuint64_t dims[1] = {(cuuint64_t)e.nl[0] * e.nl[1] * e.nl[2]};
  const cuuint64_t strides[1] = {8};
  const cuuint32_t box[1] = {(cuuint32_t)G::RXS};
  const cuuint32_t es[1] = {1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, (void*)U, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("tensor map encode failed %d\n", (int)r);
    exit(5);
  }
  if (first) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem) != cudaSuccess) exit(3);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    printf("xyz <%d,%d,%d,%d,%d>: %d regs, %zu B smem, %d B local, RXS %d\n", P, XYZ_EX, XYZ_EY, XYZ_NT, XYZ_MINB,
           fa.numRegs, G::smem, (int)fa.localSizeBytes, G::RXS);
  }
  e.ezl = XYZ_EZL;
  e.tg[0] = (e.N[0] + XYZ_EX - 1) / XYZ_EX;
  e.tg[1] = (e.N[1] + XYZ_EY - 1) / XYZ_EY;
  e.ntiles = e.tg[0] * e.tg[1] * ((e.N[2] + e.ezl - 1) / e.ezl);
  k<<<e.ntiles, XYZ_NT, G::smem, st>>>(map, U, out, out, nt, e, flag);
}
}  // namespace xyz
#define WITH_V2
#define CAND xyz
#elif defined(WITH_V2T)   // v2 with TMA row staging: scripts/experiments/explicit3d_v2_tma.cuh (measured slower)
#include <cudaTypedefs.h>
#define WITH_V2
namespace v2t {
template <int P>
void launch(const double* U, double* out, const uint8_t* nt, ExpP e, int* flag, cudaStream_t st, bool first) {
  constexpr int EX = V2_EX, EY = V2_EY;
  constexpr size_t sm = v2::smem3<P, EX, EY, true>();
  auto k = v2::k_exp3t<P, EX, EY, V2_NT, V2_MINB>;
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess || !enc)
      exit(4);
  }
  CUtensorMap map;
  const cuuint64_t dims[1] = {(cuuint64_t)e.nl[0] * e.nl[1] * e.nl[2]};
  const cuuint64_t strides[1] = {8};
  const cuuint32_t box[1] = {(cuuint32_t)v2::tma_row3<P, EX>()};
  const cuuint32_t es[1] = {1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, (void*)U, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    exit(5);
  if (first) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) exit(3);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    printf("v2t <%d,%d,%d,%d,%d>: %d regs, %zu B smem, %d B local\n", P, EX, EY, V2_NT, V2_MINB, fa.numRegs, sm,
           (int)fa.localSizeBytes);
  }
  e.ezl = V2_EZL;
  e.tg[0] = (e.N[0] + EX - 1) / EX;
  e.tg[1] = (e.N[1] + EY - 1) / EY;
  e.ntiles = e.tg[0] * e.tg[1] * ((e.N[2] + e.ezl - 1) / e.ezl);
  k<<<e.ntiles, V2_NT, sm, st>>>(map, U, out, out, nt, e, flag);
}
}  // namespace v2t
#define CAND v2t
#else
#define CAND v2
#endif

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

static void legendre(int n, double x, double& P, double& dP) {
  double p0 = 1, p1 = x;
  if (n == 0) { P = 1; dP = 0; return; }
  for (int k = 2; k <= n; ++k) {
    const double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  P = p1;
  dP = n * (x * p1 - p0) / (x * x - 1);
}

static void gauss(int n, std::vector<double>& x, std::vector<double>& w) {
  x.resize(n);
  w.resize(n);
  for (int i = 0; i < n; ++i) {
    double z = cos(M_PI * (i + 0.75) / (n + 0.5)), P, dP;
    for (int it = 0; it < 100; ++it) {
      legendre(n, z, P, dP);
      z -= P / dP;
    }
    legendre(n, z, P, dP);
    x[n - 1 - i] = z;
    w[n - 1 - i] = 2 / ((1 - z * z) * dP * dP);
  }
}

static void gll(int p, std::vector<double>& x, std::vector<double>& w) {
  x.assign(p + 1, 0);
  w.assign(p + 1, 0);
  x[0] = -1;
  x[p] = 1;
  for (int i = 1; i < p; ++i) {
    double z = -cos(M_PI * i / p);
    for (int it = 0; it < 200; ++it) {   // roots of P'_p: Newton on (1-z^2)P'_p
      double P, dP;
      legendre(p, z, P, dP);
      const double f = (1 - z * z) * dP;   // = p (P_{p-1} - z P_p)
      const double df = -p * (p + 1) * P;  // d/dz of (1-z^2)P'_p
      z -= f / df;
    }
    x[i] = z;
  }
  for (int i = 0; i <= p; ++i) {
    double P, dP;
    legendre(p, x[i], P, dP);
    w[i] = 2.0 / (p * (p + 1) * P * P);
  }
}

static void lagr(const std::vector<double>& nd, double xi, double* v, double* dv) {
  const int n = (int)nd.size();
  for (int i = 0; i < n; ++i) {
    double num = 1, den = 1, d = 0;
    for (int j = 0; j < n; ++j)
      if (j != i) {
        num *= xi - nd[j];
        den *= nd[i] - nd[j];
      }
    for (int k = 0; k < n; ++k) {
      if (k == i) continue;
      double t = 1;
      for (int j = 0; j < n; ++j)
        if (j != i && j != k) t *= xi - nd[j];
      d += t;
    }
    v[i] = num / den;
    dv[i] = d / den;
  }
}

__global__ void k_fill(double* a, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull ^ ((unsigned long long)seed << 32);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    a[i] = (double)(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}

__global__ void k_diff(const double* a, const double* b, size_t n, double* out) {
  double m = 0, r = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    m = fmax(m, fabs(a[i] - b[i]));
    r = fmax(r, fabs(a[i]));
  }
  for (int o = 16; o; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(~0u, m, o));
    r = fmax(r, __shfl_xor_sync(~0u, r, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax((unsigned long long*)out, __double_as_longlong(m));
    atomicMax((unsigned long long*)out + 1, __double_as_longlong(r));
  }
}

int main(int argc, char** argv) {
#ifndef HP
#define HP 4
#endif
  constexpr int P = HP;   // element order (compile time: -DHP=3)
  const int Ncell = argc > 1 ? atoi(argv[1]) : 160;
  const int reps = argc > 2 ? atoi(argv[2]) : 10;
  const int mask = argc > 3 ? atoi(argv[3]) : 0;
  const int Nx = argc > 4 ? atoi(argv[4]) : Ncell, Ny = argc > 5 ? atoi(argv[5]) : Ncell;
  std::vector<double> gx, gw, lx, lw;
  gauss(P + 1, gx, gw);
  gll(P, lx, lw);
  double Mh[(P + 1) * (P + 1)] = {0}, Kh[(P + 1) * (P + 1)] = {0};
  for (int q = 0; q <= P; ++q) {
    double v[P + 1], dv[P + 1];
    lagr(lx, gx[q], v, dv);
    for (int i = 0; i <= P; ++i)
      for (int j = 0; j <= P; ++j) {
        Mh[i * (P + 1) + j] += gw[q] * v[i] * v[j];
        Kh[i * (P + 1) + j] += gw[q] * dv[i] * dv[j];
      }
  }
  double iw[SC_MAXP1] = {0};
  for (int i = 0; i <= P; ++i) iw[i] = 1.0 / lw[i];
  const double iw2 = 1.0 / (lw[0] + lw[P]);
  CK(cudaMemcpyToSymbol(c_Mh, Mh, sizeof(Mh)));
  CK(cudaMemcpyToSymbol(c_Kh, Kh, sizeof(Kh)));
  CK(cudaMemcpyToSymbol(c_iw, iw, sizeof(iw)));
  CK(cudaMemcpyToSymbol(c_iw2, &iw2, sizeof(double)));
  CK(cudaMemcpyToSymbol(c_w, lw.data(), sizeof(double) * (P + 1)));
#ifdef WITH_V2
  {
    double eo[4 * SC_EO_STRIDE];
    v2::eo_blocks(P, Mh, Kh, eo);
    CK(cudaMemcpyToSymbol(c_EO, eo, sizeof(eo)));
  }
#endif

  ExpP e{};
  const int Nz = Ncell;
  e.N[0] = Nx;
  e.N[1] = Ny;
  e.N[2] = Nz;
  for (int k = 0; k < 3; ++k) {
    e.nl[k] = e.N[k] * P + 1;
    const double h = 1.0 / e.N[k];
    e.s[k] = (2 / h) * (2 / h);
  }
  e.a1 = 2;
  e.a2 = -1;
  const double dt = 0.2 / (Ncell * P * P);
  e.coefR = dt * dt;
  e.want = WANT_FAR;
  e.tiles = nullptr;
  e.clean = nullptr;
  const size_t n = (size_t)e.nl[0] * e.nl[1] * e.nl[2];
  printf("lattice %d x %d x %d (%zu nodes), p=%d\n", e.nl[0], e.nl[1], e.nl[2], n, P);
  double *U, *Pv, *O1, *O2, *dd;
  uint8_t* nt;
  CK(cudaMalloc(&U, n * 8));
  CK(cudaMalloc(&Pv, n * 8));
  CK(cudaMalloc(&O1, n * 8));
  CK(cudaMalloc(&O2, n * 8));
  CK(cudaMalloc(&nt, n));
  CK(cudaMalloc(&dd, 16));
  k_fill<<<1184, 256>>>(U, n, 1);
  k_fill<<<1184, 256>>>(Pv, n, 2);
  {
    std::vector<uint8_t> h(n, 1);
    if (mask) {
      unsigned s = 12345;
      for (size_t i = 0; i < n; ++i) {
        s = s * 1664525u + 1013904223u;
        if ((s >> 24) < 8) h[i] = 0;   // ~3% of the nodes not wanted (left untouched)
      }
    }
    CK(cudaMemcpy(nt, h.data(), n, cudaMemcpyHostToDevice));
  }
  if (!mask) {   // every tile clean (all nodes wanted): the clean-tile paths of both kernels
    uint8_t* cl;
    const size_t nt_max = (size_t)(Nx + 1) * (Ny + 1) * (Nz + 1);
    CK(cudaMalloc(&cl, nt_max));
    CK(cudaMemset(cl, 1, nt_max));
    e.clean = cl;
  }
  int* flag;
  CK(cudaMalloc(&flag, 4));
  CK(cudaMemset(flag, 0, 4));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));

  // ---- product kernel
  using T = Tile3<P>;
  ExpP e1 = e;
  e1.ezl = 16;
  e1.tg[0] = (Nx + T::E - 1) / T::E;
  e1.tg[1] = (Ny + T::EY - 1) / T::EY;
  const int tz1 = (Nz + e1.ezl - 1) / e1.ezl;
  e1.ntiles = e1.tg[0] * e1.tg[1] * tz1;
  auto k1 = k_explicit_3d<P, T::E, T::EY, T::NT, T::MINB, T::SPV>;
  CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::smem));
  auto run1 = [&](double* out) { k1<<<e1.ntiles, T::NT, T::smem>>>(U, out, out, nt, e1, flag); };
  CK(cudaMemcpy(O1, Pv, n * 8, cudaMemcpyDeviceToDevice));
  run1(O1);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float ms1 = 0;
  {
    CK(cudaMemcpy(O2, Pv, n * 8, cudaMemcpyDeviceToDevice));
    run1(O2);
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; ++r) run1(O2);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms1, a, b));
    ms1 /= reps;
  }
  {
    int hf = 0;
    CK(cudaMemcpy(&hf, flag, 4, cudaMemcpyDeviceToHost));
    printf("flag after product %d\n", hf);
  }
  printf("product k_explicit_3d<4,%d,%d,%d>: %.4f ms  (%.1f GB/s on 24 B/node)\n", T::E, T::EY, T::NT, ms1,
         24.0 * n / ms1 / 1e6);
#ifdef WITH_V2
  CK(cudaMemcpy(O2, Pv, n * 8, cudaMemcpyDeviceToDevice));
  CAND::launch<P>(U, O2, nt, e, flag, 0, true);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(dd, 0, 16));
  k_diff<<<1184, 256>>>(O1, O2, n, dd);
  double hd[2];
  CK(cudaMemcpy(hd, dd, 16, cudaMemcpyDeviceToHost));
  printf("cand vs product: max|diff| = %.3e, max|out| = %.3e, rel %.3e\n", hd[1] > 0 ? hd[0] : 0.0, hd[1],
         hd[0] / hd[1]);
  if (n < 4000000) {   // small lattices: where do the two kernels differ
    std::vector<double> h1(n), h2(n);
    CK(cudaMemcpy(h1.data(), O1, n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), O2, n * 8, cudaMemcpyDeviceToHost));
    int shown = 0;
    size_t bad = 0;
    for (size_t g = 0; g < n; ++g)
      if (fabs(h1[g] - h2[g]) > 1e-12 * (1 + fabs(h1[g]))) {
        ++bad;
        if (shown < 25) {
          const int i = g % e.nl[0], j = (g / e.nl[0]) % e.nl[1], k = g / ((size_t)e.nl[0] * e.nl[1]);
          printf("  diff at (%d,%d,%d): %.6e vs %.6e\n", i, j, k, h1[g], h2[g]);
          ++shown;
        }
      }
    printf("  %zu differing nodes of %zu\n", bad, n);
    std::vector<int> pk(e.nl[2], 0), py(e.nl[1], 0), px(e.nl[0], 0);
    for (size_t g = 0; g < n; ++g)
      if (fabs(h1[g] - h2[g]) > 1e-12 * (1 + fabs(h1[g]))) {
        px[g % e.nl[0]]++;
        py[(g / e.nl[0]) % e.nl[1]]++;
        pk[g / ((size_t)e.nl[0] * e.nl[1])]++;
      }
    printf("  per z:");
    for (int k = 0; k < e.nl[2]; ++k) printf(" %d", pk[k]);
    printf("\n  per y:");
    for (int k = 0; k < e.nl[1]; ++k) printf(" %d", py[k]);
    printf("\n  per x:");
    for (int k = 0; k < e.nl[0]; ++k) printf(" %d", px[k]);
    printf("\n");
  }
  float ms2 = 0;
  {
    CAND::launch<P>(U, O2, nt, e, flag, 0, false);
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; ++r) CAND::launch<P>(U, O2, nt, e, flag, 0, false);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms2, a, b));
    ms2 /= reps;
  }
  printf("cand: %.4f ms  (%.1f GB/s on 24 B/node)\n", ms2, 24.0 * n / ms2 / 1e6);
#endif
  int hf = 0;
  CK(cudaMemcpy(&hf, flag, 4, cudaMemcpyDeviceToHost));
  printf("flag %d\n", hf);
  return 0;
}
