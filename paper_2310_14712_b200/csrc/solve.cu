// (a5) implicit cut-DOF solve S a^c_{n+1} = r^c with the factor computed once at setup
// ("triangular matrix system with the factorized system
// matrix S" each step).  The factor is of the Jacobi-scaled matrix D S D (factor.cpp).
//
// Supernodal block substitution with each supernode's triangular solves folded into its
// panel (factor.cpp make_panel): with L = [L_ss 0; L_Rs L_RR],
//   forward   v_s = b_s - (updates of the children),  q_s = D_s v_s,  U_s = G_s v_s (+ children)
//   backward  x_s = q_s - G_s^T x_R
// where D_s = (L_ss L_ss^T)^{-1} and G_s = L_Rs L_ss^{-1}; this equals L_ss^{-T}(L_ss^{-1} v_s
// - L_Rs^T x_R), i.e. the two triangular solves of the block algorithm, so each supernode has
// ONE dependent phase per sweep (the critical path is the elimination-tree height, once per
// sweep) and one stacked GEMV [D_s; G_s] v_s per forward phase.
//
// One persistent kernel performs both sweeps, driven by a READY QUEUE of work items: the
// forward items of the leaves are ready at launch; the CTA that completes the last block of a
// phase pushes the items that this completion makes ready (forward of the parent once all its
// children are done; backward of the root after its forward; backward of the children after a
// backward).  A CTA therefore only ever holds a ready item: no CTA waits on dependencies while
// holding an item, all resident CTAs work.  Per item: take the next queue slot, stream the
// item's panel tile into shared memory with bulk (TMA) copies completing on an mbarrier,
// gather the produced vector entries meanwhile, contract, publish.
// Tiles: forward 32*2^k panel rows x <= SOLVE_TILE columns, backward <= 32 outputs x <=
// SOLVE_BROWS rows.  A block whose reduction spans several tiles writes per-tile partials; the
// publisher of the LAST tile (atomic ticket) sums them in fixed tile order -> deterministic
// results regardless of the schedule.
// Small supernodes (whole panel <= one staging buffer) are one item per phase.
// CTA roles (warp specialisation, k_solve below): a claimer warp takes queue slots and issues
// the panel copies, 4 compute warps gather / contract / emit, a publisher warp draws tile
// tickets, sums partials and publishes completions (fences, counters, pushes).
// Progress: a slot that may still be empty is only awaited by a CTA whose compute warps hold
// no item (a CTA claims ahead of its current item only when the queue backlog exceeds one
// item per CTA, so that slot is already pushed); if every CTA waits, every pushed item is
// finished and its completion pushed its dependents, so the queue advances until all n_items
// slots are filled.  Publication: results, fence.acq_rel, counter atomics
// (release); the pusher fences after observing the final count and then stores the slots
// (fence + relaxed store = release); the consumer acquire-loads the slot.
#include <cstdlib>

#include "sc_internal.h"

namespace {

enum { IT_F = 0, IT_B = 1 };
// SC_TRACE_COMPUTE (experiment builds): the trace records the compute warps' chain instead —
// [READY passed, gathered, staged, contracted, record slot free]
#ifdef SC_TRACE_COMPUTE
#define TRC(k) if (a.trace && tid == 0) a.trace[5 * (size_t)it + (k)] = gtimer()
#else
#define TRC(k)
#endif
constexpr int NT = SOLVE_NT;          // threads per CTA
constexpr int NWC = NT / 32 - 2;      // compute warps (then the claimer and publisher warps)
constexpr int NTC = NWC * 32;
static_assert(NWC * 8 >= 32, "backward tiles: <= 32 columns, <= 8 per compute warp");
constexpr int VS = SOLVE_BROWS > SOLVE_TILE + NTC ? SOLVE_BROWS : SOLVE_TILE + NTC;   // gathered vector

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// release / acquire fence at GPU scope (fence.acq_rel: the publication patterns here are
// release -> relaxed RMW/store and relaxed RMW -> acquire; no SC fence is needed)
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// push cnt items starting at first (warp; the caller fenced after observing the completion
// it reacts to, so relaxed slot stores publish everything before the fence)
__device__ __forceinline__ void push_items(const SolveDev& a, int first, int cnt, int lane) {
  int slot = 0;
  if (lane == 0 && cnt) slot = atomicAdd(a.tail, cnt);
  slot = __shfl_sync(0xffffffffu, slot, 0);
  for (int k = lane; k < cnt; k += 32) st_relaxed(a.ready + slot + k, first + k + 1);
}

// one block of phase ph of supernode s is published (publisher warp, after the block's
// results were written); the warp completing the phase pushes its dependents.  The item
// ranges of the dependents (read-only metadata) are loaded by all lanes BEFORE lane 0's
// fence and atomics, so they are not on the publication's dependent-latency chain; the
// backward children are pushed with one tail reservation for all of them.
__device__ __forceinline__ void complete_block(const SolveDev& a, int ph, int s, int lane) {
  const int n_sn = a.n_sn;
  int pf = 0, pc = 0, nchp = 0, p = -1;      // forward: the parent's (or own backward) range
  int ch0 = 0, nchl = 0, cf = 0, cc = 0;     // backward: children (lane q: child q)
  if (ph == 0) {
    p = a.parent[s];
    const int ps = p >= 0 ? p : n_sn + s;
    pf = a.item_first[ps];
    pc = a.item_cnt[ps];
    if (p >= 0) nchp = a.nch[p];
  } else {
    ch0 = a.chptr[s];
    nchl = a.chptr[s + 1] - ch0;
    if (lane < nchl) {
      const int ch = a.chidx[ch0 + lane];
      cf = a.item_first[n_sn + ch];
      cc = a.item_cnt[n_sn + ch];
    }
  }
  const int nb = a.nblk[ph * n_sn + s];
  int act = 0;   // 0 nothing, 1 phase complete (forward: 2 parent ready, 3 root)
  if (lane == 0) {
    fence_acq_rel();   // release: the compute warps' results (ordered before DONE)
    // a single-block phase / a single child needs no counter: this block completes it.  After
    // an observed counter, one fence acquires the other blocks' results and releases them to
    // the next counter / the pushed slots.
    bool done = true;
    if (nb > 1) {
      done = atomicAdd(a.cnt + ph * n_sn + s, 1) == nb - 1;
      if (done) fence_acq_rel();
    }
    if (done) {
      act = 1;
      if (ph == 0) {
        if (p < 0) {
          act = 3;
        } else if (nchp == 1) {
          act = 2;
        } else if (atomicAdd(a.done_ch + p, 1) == nchp - 1) {
          fence_acq_rel();
          act = 2;
        }
      }
    }
  }
  act = __shfl_sync(0xffffffffu, act, 0);
  if (!act) return;
  if (ph == 0) {
    if (act >= 2) push_items(a, pf, pc, lane);   // parent forward (2) or own backward (3)
    return;
  }
  for (int base = 0; base < nchl; base += 32) {
    if (base > 0) {   // more than 32 children (not produced by the bisection ordering)
      cf = cc = 0;
      if (base + lane < nchl) {
        const int ch = a.chidx[ch0 + base + lane];
        cf = a.item_first[n_sn + ch];
        cc = a.item_cnt[n_sn + ch];
      }
    }
    int incl = cc;   // inclusive scan of the children's item counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int slot = 0;
    if (lane == 0 && total) slot = atomicAdd(a.tail, total);
    slot = __shfl_sync(0xffffffffu, slot, 0) + incl - cc;
    for (int k = 0; k < cc; ++k) st_relaxed(a.ready + slot + k, cf + k + 1);
  }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
// global -> shared bulk copy (TMA engine); bytes and both addresses multiples of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

struct Item {
  int type, s, t, ntb, pslot, bctr, r0, nr, c0, nc;   // see factor.cpp (fat items)
  int dof0, w, r, goff, uoff, roff, ld, wp;
  int64_t aoff;
};

// the item in queue slot h (waits until the slot is filled); -1 past the end
__device__ __forceinline__ int slot_item(const SolveDev& a, int h) {
  if (h >= a.n_items) return -1;
  if (h < a.n_init) return a.init[h];
  const int* slot = a.ready + (h - a.n_init);
  int v;
  unsigned ns = 32;
  while ((v = ld_acquire(slot)) == 0) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
  return v - 1;
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// copy item it's 80-byte descriptor to shared memory (one thread)
__device__ __forceinline__ void fetch_desc(const SolveDev& a, int it, int4* dst) {
  const int4* d = a.items + 5 * (size_t)it;
#pragma unroll
  for (int k = 0; k < 5; ++k) dst[k] = d[k];
}

// sum of the children's update entries at front position t (inline list, else CSR)
__device__ __forceinline__ double child_sum(const SolveDev& a, int t) {
  const int2 g = a.g2[t];
  if (g.x >= 0) {
    double v = __ldcg(a.U + g.x);
    if (g.y >= 0) v += __ldcg(a.U + g.y);
    return v;
  }
  double v = 0.0;
  if (g.x <= -2)
    for (int q = -2 - g.x; q < a.gptr[t + 1]; ++q) v += __ldcg(a.U + a.gidx[q]);
  return v;
}

__device__ __forceinline__ Item load_item(const int4* d) {
  const int4 d0 = d[0], d1 = d[1], d2 = d[2], d3 = d[3], d4 = d[4];
  Item m;
  m.type = d0.x;
  m.s = d0.y;
  m.t = d0.z;
  m.ntb = d0.w;
  m.pslot = d1.x;
  m.bctr = d1.y;
  m.r0 = d1.z;
  m.nr = d1.w;
  m.c0 = d2.x;
  m.nc = d2.y;
  m.dof0 = d2.z;
  m.w = d2.w;
  m.r = d3.x;
  m.goff = d3.y;
  m.uoff = d3.z;
  m.roff = d3.w;
  m.aoff = (int64_t)(uint32_t)d4.x | ((int64_t)d4.y << 32);
  m.ld = d4.z;
  m.wp = d4.w;
  return m;
}

// issue the bulk copies of item m's panel tile into `st` (warp 0): one column segment per
// staged column; lane 0 arms `bar` with the byte count first.  Staged layout: column j of
// the tile at st + j * nr (F: panel rows r0.., B: G rows r0..).
__device__ __forceinline__ void stage_item(const SolveDev& a, const Item& m, double* st, uint64_t* bar, int lane) {
  const double* Ap = a.A + m.aoff;
  const int nr = m.nr;
  if (lane == 0) mbar_expect(bar, (unsigned)(m.nc * nr * 8));
  __syncwarp();
  if (nr == 0) return;
  const size_t row0 = (m.type == IT_F) ? (size_t)m.r0 : (size_t)m.wp + m.r0;
  if (row0 == 0 && nr == m.ld) {   // whole columns: the tile is one contiguous range
    if (lane == 0) bulk_g2s(st, Ap + (size_t)m.c0 * m.ld, (unsigned)(m.nc * nr * 8), bar);
    return;
  }
  for (int j = lane; j < m.nc; j += 32)
    bulk_g2s(st + j * nr, Ap + (size_t)(m.c0 + j) * m.ld + row0, nr * 8, bar);
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// named barriers: READY (claimer -> compute: next item's descriptor in smem, its copy issued),
// FREE (compute -> claimer: staging buffer consumed), DONE+b (compute -> publisher: the item
// whose completion record is in s_pub[b] is written), CONS+b (publisher -> compute: s_pub[b]
// consumed), CB (compute warps only).  Two records so the compute warps can run one item ahead
// of the publisher.
enum { BAR_READY = 1, BAR_FREE = 2, BAR_DONE = 3, BAR_CONS = 5, BAR_CB = 7 };
constexpr int NTX = NTC + 32;   // threads taking part in a compute <-> control-warp barrier

// claimer warp: take the next queue slot, stage its descriptor into dst (lane 0); returns the
// item (-1 past the end), broadcast to the warp
__device__ __forceinline__ int claim(const SolveDev& a, int4* dst, int* s_it, int lane) {
  int it = 0;
  if (lane == 0) {
    const unsigned long long t0 = a.trace ? gtimer() : 0;
    it = slot_item(a, atomicAdd(a.head, 1));
    if (it >= 0) fetch_desc(a, it, dst);
    *s_it = it;
#ifdef SC_TRACE_COMPUTE
    if (false) {
#else
    if (a.trace && it >= 0) {
#endif
      a.trace[5 * (size_t)it] = t0;
      a.trace[5 * (size_t)it + 1] = gtimer();
    }
  }
  return __shfl_sync(0xffffffffu, it, 0);
}

// publisher warp, record of a tile of a multi-tile group (its partials written and ordered
// before DONE): draw the group's ticket; the LAST tile's publisher sums the ntb partials in
// tile order (deterministic) and emits the group's outputs — forward: q_s rows / U_s rows
// (+ the children's update entries), backward: x_s = q_s - G_s^T x_R.  Returns whether this
// tile completed its group (the caller then publishes the block).
__device__ __forceinline__ bool tile_ticket(const SolveDev& a, int it, int lane) {
  int4 d[5];
  const int4* src = a.items + 5 * (size_t)it;
#pragma unroll
  for (int k = 0; k < 5; ++k) d[k] = src[k];
  const Item m = load_item(d);
  int last = 0;
  if (lane == 0) {
    fence_acq_rel();   // release this tile's partials
    last = atomicAdd(a.bcnt + m.bctr, 1) == m.ntb - 1;
    if (last) fence_acq_rel();   // acquire the other tiles' partials
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return false;
  const double* P = a.part + m.pslot;
  if (m.type == IT_F) {
    for (int o = lane; o < m.nr; o += 32) {
      double v = 0.0;
      for (int k = 0; k < m.ntb; ++k) v += __ldcg(P + k * m.nr + o);
      const int i = m.r0 + o;
      if (i < m.w) {
        a.q[m.dof0 + i] = v;
      } else if (i >= m.wp && i < m.wp + m.r) {
        const int k = i - m.wp;
        a.U[m.uoff + k] = v + child_sum(a, m.goff + m.w + k);
      }
    }
  } else {
    for (int o = lane; o < m.nc; o += 32) {
      double v = 0.0;
      for (int k = 0; k < m.ntb; ++k) v += __ldcg(P + k * 32 + o);
      const int j = m.c0 + o;
      if (j < m.w) a.x[m.dof0 + j] = __ldcg(a.q + m.dof0 + j) - v;
    }
  }
  __syncwarp();   // the lanes' emits precede lane 0's releasing fence in complete_block
  return true;
}

// Warp-specialised persistent CTA: NWC compute warps gather and contract the staged tiles; a
// claimer warp takes items from the queue and issues their panel copies; a publisher warp
// publishes completions.  The three chains (claim latency, contraction, publication fences and
// atomics) overlap across consecutive items of the CTA.
__global__ void __launch_bounds__(NT, SOLVE_MINB) k_solve(SolveDev a) {   // CTAs/SM (shared memory)
  extern __shared__ __align__(128) double stg[];   // c->solve_stage doubles (factor.cpp)
  __shared__ double vs[VS];
  double* red = vs + SOLVE_TILE;   // forward reductions (the gathered vector has <= SOLVE_TILE entries)
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int s_it[2], s_off[2];
  __shared__ int4 s_desc[2][5];
  __shared__ int4 s_pub[2];   // completion records: item, type, supernode, 1 single tile / 2 tile of a group
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar[0]);
    mbar_init(&bar[1]);
  }
  __syncthreads();
  if (warp == NWC) {
    // ---------------- claimer warp ----------------
    // Item k is staged at offset s_off[k & 1] of the staging buffer and completes on mbarrier
    // bar[k & 1].  In the throughput regime the next item is claimed while item k is
    // contracted, and its copy is issued at once if it fits beside item k (after it, or before
    // it from offset 0); otherwise after FREE (item k contracted).  Each iteration consumes
    // exactly one FREE (item k's) before READY(k+1), so READY runs at most one item ahead of
    // the compute warps and only item k can be live in the buffer.
    const int STG = a.stage;
    int buf = 0, off = 0, size = 0;
    int it = claim(a, s_desc[0], &s_it[0], lane);
    if (it >= 0) {
      const Item m0 = load_item(s_desc[0]);
      size = m0.nc * m0.nr;
      if (lane == 0) s_off[0] = 0;
      stage_item(a, m0, stg, &bar[0], lane);
    }
    named_arrive(BAR_READY, NTX);
    while (it >= 0) {
      const int nb = buf ^ 1;
      // claim ahead when the queue backlog exceeds one item per CTA; otherwise only once the
      // compute warps are free, so a latency-bound solve never parks a ready item behind a
      // busy CTA
      int ahead = 0;
      if (lane == 0) ahead = a.n_init + ld_relaxed(a.tail) > ld_relaxed(a.head) + (int)gridDim.x;
      bool freed = false;
      if (!__shfl_sync(0xffffffffu, ahead, 0)) {
        named_sync(BAR_FREE, NTX);
        freed = true;
      }
      const int nx = claim(a, s_desc[nb], &s_it[nb], lane);
      if (nx >= 0) {
        const Item mn = load_item(s_desc[nb]);
        const int nsize = mn.nc * mn.nr;
        int noff = 0;
        if (!freed) {
          if (off + size + nsize <= STG) {
            noff = off + size;
          } else if (nsize > off) {   // fits nowhere beside item k: wait until it is contracted
            named_sync(BAR_FREE, NTX);
            freed = true;
          }
        }
        if (lane == 0) s_off[nb] = noff;
        stage_item(a, mn, stg + noff, &bar[nb], lane);
        off = noff;
        size = nsize;
      }
      if (!freed) named_sync(BAR_FREE, NTX);
      named_arrive(BAR_READY, NTX);
      buf = nb;
      it = nx;
    }
    return;
  }
  if (warp == NWC + 1) {
    // ---------------- publisher warp ----------------
    named_arrive(BAR_CONS, NTX);
    named_arrive(BAR_CONS + 1, NTX);
    for (int buf = 0;; buf ^= 1) {
      if (buf) named_sync(BAR_DONE + 1, NTX);
      else named_sync(BAR_DONE, NTX);
      const int4 r = s_pub[buf];
      if (buf) named_arrive(BAR_CONS + 1, NTX);
      else named_arrive(BAR_CONS, NTX);
      if (r.x < 0) return;
      // the compute warps' result stores precede DONE; lane 0's fence is cumulative over them
      if (r.w == 2 && !tile_ticket(a, r.x, lane)) continue;   // a tile of a group, not the last
      complete_block(a, r.y == IT_F ? 0 : 1, r.z, lane);
#ifndef SC_TRACE_COMPUTE
      if (a.trace && lane == 0) a.trace[5 * (size_t)r.x + 4] = gtimer();
#endif
    }
  }
  // ---------------- compute warps (tid < NTC) ----------------
  unsigned phase = 0;   // mbarrier parity per item parity (bit b)
  for (int buf = 0, pb = 0;; buf ^= 1, pb ^= 1) {
    named_sync(BAR_READY, NTX);
    const int it = s_it[buf];
    if (it < 0) {
      if (pb) named_sync(BAR_CONS + 1, NTX);
      else named_sync(BAR_CONS, NTX);
      if (tid == 0) s_pub[pb] = make_int4(-1, 0, 0, 0);
      if (pb) named_arrive(BAR_DONE + 1, NTX);
      else named_arrive(BAR_DONE, NTX);
      return;
    }
    const Item m = load_item(s_desc[buf]);
    TRC(0);
    const double* stg_b = stg + s_off[buf];
    const bool fwd = (m.type == IT_F);
    const int go = m.goff;
    // gather the input vector while the panel copy is in flight (every producer of it
    // completed before this item was pushed; L1 bypass)
    if (fwd) {
      // v_j = b_j - sum of the children's update entries at column position j
      for (int j = tid; j < m.nc; j += NTC) {
        const int pj = m.c0 + j;
        vs[j] = a.b[m.dof0 + pj] - child_sum(a, go + pj);
      }
    } else {
      const int rr = min(m.nr, m.r - m.r0);   // real (unpadded) rows of this tile
      for (int i = tid; i < rr; i += NTC) vs[i] = __ldcg(a.x + a.R[m.roff + m.r0 + i]);
      if (tid == 0 && rr < m.nr && rr >= 0) vs[rr] = 0.0;   // padding row
    }
    // backward, single-tile group: q of the output column of lanes 4k (column warp + k NWC),
    // loaded now (off the path after the contraction); those lanes emit
    double qpre = 0.0;
    if (!fwd && m.ntb == 1 && (lane & 3) == 0) {
      const int cc = warp + (lane >> 2) * NWC;
      if (cc < m.nc && m.c0 + cc < m.w) qpre = __ldcg(a.q + m.dof0 + m.c0 + cc);
    }
    // forward: the children's contributions to the update rows this thread will emit (rows
    // r0 + tid + k NTC), gathered now so they overlap the panel copy instead of following it
    constexpr int NCR = 4;
    double crv[NCR];
#pragma unroll
    for (int k = 0; k < NCR; ++k) {
      crv[k] = 0.0;
      const int i = m.r0 + tid + k * NTC;
      if (fwd && tid + k * NTC < m.nr && i >= m.wp && i < m.wp + m.r) {
        crv[k] = child_sum(a, go + m.w + (i - m.wp));
      }
    }
#if !defined(SC_TRACE_COMPUTED) && !defined(SC_TRACE_COMPUTE)
    if (a.trace && tid == 0) a.trace[5 * (size_t)it + 2] = gtimer();
#endif
    TRC(1);
    while (!mbar_try(&bar[buf], (phase >> buf) & 1)) {
    }
    phase ^= 1u << buf;
#ifndef SC_TRACE_COMPUTE
    if (a.trace && tid == 0) a.trace[5 * (size_t)it + 3] = gtimer();
#endif
    TRC(2);
    named_sync(BAR_CB, NTC);   // vs complete
    // panel row i (= r0 + tid + kq NTC) of the forward phase -> q_s or U_s
    auto emit_f = [&](int i, double v, int kq) {
      if (i < m.w) {
        a.q[m.dof0 + i] = v;
      } else if (i >= m.wp && i < m.wp + m.r) {
        const int k = i - m.wp;
        if (kq < NCR) {
#pragma unroll
          for (int t = 0; t < NCR; ++t)
            if (t == kq) v += crv[t];
        } else {
          v += child_sum(a, go + m.w + k);
        }
        a.U[m.uoff + k] = v;
      }
    };
    double* P = a.part + m.pslot;
    if (fwd) {
      // rows i of the tile: nr rows, nc columns; G threads per row when nr < NTC
      const int nr = m.nr, nc = m.nc;
      if (nr >= NTC) {
        for (int i = tid; i < nr; i += NTC) {
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;   // 4 independent chains
          int j = 0;
          for (; j + 3 < nc; j += 4) {
            a0 += stg_b[j * nr + i] * vs[j];
            a1 += stg_b[(j + 1) * nr + i] * vs[j + 1];
            a2 += stg_b[(j + 2) * nr + i] * vs[j + 2];
            a3 += stg_b[(j + 3) * nr + i] * vs[j + 3];
          }
          for (; j < nc; ++j) a0 += stg_b[j * nr + i] * vs[j];
          const double v = (a0 + a1) + (a2 + a3);
          if (m.ntb == 1) emit_f(m.r0 + i, v, (i - tid) / NTC);
          else P[m.t * nr + i] = v;
        }
        named_arrive(BAR_FREE, NTX);
      } else {
        const int G = NTC / nr;   // nr >= 2
        const int i = tid % nr, g = tid / nr;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;   // 4 independent chains
        if (g < G) {
          int j = g;
          for (; j + 3 * G < nc; j += 4 * G) {
            a0 += stg_b[j * nr + i] * vs[j];
            a1 += stg_b[(j + G) * nr + i] * vs[j + G];
            a2 += stg_b[(j + 2 * G) * nr + i] * vs[j + 2 * G];
            a3 += stg_b[(j + 3 * G) * nr + i] * vs[j + 3 * G];
          }
          for (; j < nc; j += G) a0 += stg_b[j * nr + i] * vs[j];
        }
        red[tid] = (a0 + a1) + (a2 + a3);
        named_arrive(BAR_FREE, NTX);
        named_sync(BAR_CB, NTC);
        if (tid < nr) {
          double v = 0.0;
          for (int k = 0; k < G; ++k) v += red[k * nr + tid];
          if (m.ntb == 1) emit_f(m.r0 + tid, v, 0);
          else P[m.t * nr + tid] = v;
        }
      }
    } else {
      // outputs: nc <= 32 columns of G_s; warp w handles columns w + k NWC (k < 8) all at once
      // (one vs load per row, 8 independent chains), lanes stride rows; a transposing
      // butterfly (9 shuffles) leaves column k's sum in lanes 4k .. 4k+3
      const int nr = m.nr;
      double acc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0.0;
      for (int i = lane; i < nr; i += 32) {
        const double v = vs[i];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int cc = warp + k * NWC;
          if (cc < m.nc) acc[k] += stg_b[cc * nr + i] * v;
        }
      }
      const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
      double r4[4], r2[2];
#pragma unroll
      for (int t = 0; t < 4; ++t)
        r4[t] = (h16 ? acc[t + 4] : acc[t]) + __shfl_xor_sync(0xffffffffu, h16 ? acc[t] : acc[t + 4], 16);
#pragma unroll
      for (int t = 0; t < 2; ++t)
        r2[t] = (h8 ? r4[t + 2] : r4[t]) + __shfl_xor_sync(0xffffffffu, h8 ? r4[t] : r4[t + 2], 8);
      double v = (h4 ? r2[1] : r2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? r2[0] : r2[1], 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      const int cc = warp + (lane >> 2) * NWC;   // this lane's column (lanes 4k .. 4k+3: column k)
      if ((lane & 3) == 0 && cc < m.nc) {
        if (m.ntb == 1) {
          if (m.c0 + cc < m.w) a.x[m.dof0 + m.c0 + cc] = qpre - v;
        } else {
          P[m.t * 32 + cc] = v;
        }
      }
      named_arrive(BAR_FREE, NTX);
    }
    TRC(3);
    // completion record for the publisher (its fence is cumulative over the compute warps'
    // result stores ordered before DONE); wait until the record slot is free
    if (pb) named_sync(BAR_CONS + 1, NTX);
    else named_sync(BAR_CONS, NTX);
    TRC(4);
    if (tid == 0) s_pub[pb] = make_int4(it, m.type, m.s, m.ntb > 1 ? 2 : 1);
#ifdef SC_TRACE_COMPUTED
    if (a.trace && tid == 0) a.trace[5 * (size_t)it + 2] = gtimer();   // experiment: compute done
#endif
    if (pb) named_arrive(BAR_DONE + 1, NTX);
    else named_arrive(BAR_DONE, NTX);
  }
}

}  // namespace

void launch_solve(sc_ctx* c, const Factor& f, cudaStream_t st) {
  if (c->n_cl == 0 || c->n_items == 0) return;
  SolveDev a = c->solve_dev;
  a.A = f.A;
  const int smem = (int)(sizeof(double) * c->solve_stage);
  if (c->solve_grid == 0) {
    SC_CUDA(cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    SC_CUDA(cudaFuncSetAttribute(k_solve, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int per_sm = 0, sms = 0, dev = 0;
    SC_CUDA(cudaGetDevice(&dev));
    SC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve, NT, smem));
    // cap the resident solve CTAs (room for the concurrent far-d update, step.cu)
    int cap = c->solve_cap;
    if (const char* v = sc_knob("SC_SOLVE_CTAS_PER_SM")) cap = atoi(v);
    if (cap > 0) per_sm = std::max(1, std::min(per_sm, cap));
    c->solve_grid = std::max(1, std::min(c->n_items, per_sm * sms));
  }
  SC_CUDA(cudaMemsetAsync(c->d_solve_cnt, 0, sizeof(int) * c->n_counters, st));
  k_solve<<<c->solve_grid, NT, smem, st>>>(a);
  SC_CUDA(cudaGetLastError());
}
