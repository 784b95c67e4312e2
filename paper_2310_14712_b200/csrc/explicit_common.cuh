// Definitions shared by the explicit kernels of libsc (step.cu is the only translation unit of
// the library that includes this file; scripts/exp_harness.cu includes it for kernel
// experiments): the 1D reference operators in constant memory and the launch parameters.
#pragma once
#include <stdint.h>

#ifndef SC_MAXP1
#define SC_MAXP1 9
#endif

__constant__ double c_Mh[SC_MAXP1 * SC_MAXP1];
__constant__ double c_Kh[SC_MAXP1 * SC_MAXP1];
__constant__ double c_w[SC_MAXP1];
__constant__ double c_iw[SC_MAXP1];   // 1 / w_l
__constant__ double c_iw2;            // 1 / (2 w_0): interior element-boundary node

enum { WANT_FAR = 1 << 1, WANT_NEAR = 1 << 4 };

struct ExpP {
  int nl[3];
  int N[3];
  double s[3];      // (2/h_k)^2
  double a1, a2, coefR;  // out = a1 u + a2 P - coefR * r' / prod(wt)
  int want;         // bit mask of the node types updated by this launch: bit 1 tensor-d far
                    // from c nodes, bit 4 tensor-d near c nodes (WANT_FAR / WANT_NEAR)
  int tg[2];        // tile-grid extents in x, y
  int ntiles;       // tiles of this launch (blocks loop over them with a grid stride)
  const int* tiles; // nullable: tile ids (x fastest) of a tile-list launch
  const uint8_t* clean;  // nullable: per tile id, 1 = every node it owns is wanted tensor-d
  int ezl;          // 3D: element layers per tile along z
};

// tile coordinates of the tt-th tile of the launch: from the tile list if any, else linear
__device__ __forceinline__ int3 tile_of(const ExpP& e, int tt) {
  const int id = e.tiles ? e.tiles[tt] : tt;
  return make_int3(id % e.tg[0], (id / e.tg[0]) % e.tg[1], id / (e.tg[0] * e.tg[1]));
}

