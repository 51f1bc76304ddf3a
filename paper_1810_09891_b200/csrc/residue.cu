// Residue-owned gridding kernels (sm_100a) for d = 3, m = 4, 8^3 tiles:
//   B^H (spread): g[l mod n] += f_j prod_i psi_i(x_ji - l_i / n_i)   kernels.py:209-401
//   B   (interp): f_j = sum_l g[l mod n] prod_i psi_i(...)           kernels.py:122-197
//
// A regular node (stencil 2m = 8 cells wide in every dim) of an 8^3 tile
// touches the halo cells h_i .. h_i + 7 with h_i = its cell inside the tile,
// so the cells it touches lie in a 15^3 halo and cover every residue class
// (a mod 8, b mod 8) of the leading two dims exactly once.  A TEAM of 64
// lanes therefore owns the halo by residue: lane (ra, rb) holds the halo row
// (a, b, 0..14) with a = ra or ra + 8, b = rb or rb + 8 -- whichever lies in
// the current node's stencil -- as 15 complex register accumulators, and
// every lane does useful FMAs for every node (the row-per-thread kernels in
// gridding.cu keep 17^2 rows on 289 threads of which 64 work per node).
//   * Nodes of a tile arrive sorted by (h_1, then h_0 in serpentine order)
//     (k_bin_keys), so the row a lane needs changes rarely: when h_0 passes
//     ra (8 lanes of one warp, ~56 times per tile) or h_1 passes rb (7 times).
//     The leaving row goes to the lane's own slot of the team's shared-memory
//     halo, the entering one comes from there (zero if never written).
//   * Row stride 15 cells (240 B): the 8 lanes of a quarter warp (rb = 0..7)
//     hit 8 different 16-byte bank groups; no other lane touches a lane's
//     rows, so there are no atomics and no barriers in the spread.
//   * Node batches (PRE_PSI rows of 3 x 8 factors, 4-byte stencil records,
//     samples / output indices) arrive by TMA bulk copies on a per-team
//     mbarrier ring; the spread flushes each written row with one TMA bulk
//     fp64 reduction into the dense grid (periodic wrap per row); the interp
//     loads the 15^3 halo with one TMA tensor copy per tile.
//   * One persistent CTA per SM holds NT independent teams (own halo, ring,
//     barriers and subproblem tickets).
// Nodes with a 2m+1 wide stencil in some dim (n x an exact integer) are
// skipped here and handled by k_wide_* (direct window evaluation, atomics).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "async.cuh"
#include "common.cuh"
#include "kernels.h"

namespace nfftk {

struct ResMeta {
  int tile;  // tile of this batch
  int nb;    // nodes (< 0: end of work)
  int last;  // last batch of its subproblem
  int off;   // offset of the 4-byte arrays inside the stage (16-byte bulk copies)
};

template <typename R, int NT_, int NB_, int S_, bool INTERP>
struct ResCfg {
  static constexpr int NT = NT_, NB = NB_, S = S_;
  static constexpr int ELEM = 2 * (int)sizeof(R);
  static constexpr int FA = 16 / ELEM;                     // samples per 16 bytes
  static constexpr int ROW = RES_H * ELEM;                 // one halo row, bytes
  static constexpr size_t al(size_t v) { return (v + 15) & ~(size_t)15; }
  static constexpr size_t al128(size_t v) { return (v + 127) & ~(size_t)127; }
  static constexpr size_t HALO = al128((size_t)RES_H * RES_H * ROW);
  static constexpr size_t W_BYTES = al(sizeof(R) * NB * RES_PR);
  static constexpr size_t R_BYTES = al(4 * (size_t)(NB + 4));
  static constexpr size_t X_BYTES = INTERP ? al(4 * (size_t)(NB + 4)) : al((size_t)ELEM * (NB + FA));
  static constexpr size_t SB = W_BYTES + R_BYTES + X_BYTES;
  static constexpr size_t CTL = al(8 * (2 * (size_t)S + 2) + sizeof(ResMeta) * S + 32);
  static constexpr size_t PART = INTERP ? (size_t)S * 2 * NB * ELEM : 0;  // interp: per-warp node sums
  static constexpr size_t TEAM_BYTES = al128(HALO + S * SB + CTL + PART);
  static constexpr size_t SMEM = NT * TEAM_BYTES;
  static constexpr int THREADS = NT * 64;
};

template <typename R>
__device__ __forceinline__ void load8(const R* w, R* o) {
  if constexpr (sizeof(R) == 8) {
    const double2* p = reinterpret_cast<const double2*>(w);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 v = p[i];
      o[2 * i] = v.x;
      o[2 * i + 1] = v.y;
    }
  } else {
    const float4* p = reinterpret_cast<const float4*>(w);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float4 v = p[i];
      o[4 * i] = v.x;
      o[4 * i + 1] = v.y;
      o[4 * i + 2] = v.z;
      o[4 * i + 3] = v.w;
    }
  }
}

__device__ __forceinline__ void team_sync(int team) {
  asm volatile("bar.sync %0, 64;\n" ::"r"(team + 1) : "memory");
}

// Team ticket order: team t of CTA b starts at subproblem b * NT + t, then
// draws nteams + ticket from the plan's counter (common.cuh next_sub, per team).
__device__ __forceinline__ int res_next_sub(const Geom& g, int slot, int cur, int nteams) {
  if (!g.sched) return cur + nteams;
  return nteams + (int)atomicAdd(g.sched + slot, 1u);
}
__device__ __forceinline__ void res_sched_done(const Geom& g, int slot, int nteams) {
  if (!g.sched) return;
  __threadfence();
  if (atomicAdd(g.sched + slot + 1, 1u) == (unsigned)nteams - 1) {
    g.sched[slot] = 0;
    g.sched[slot + 1] = 0;
    __threadfence();
  }
}

// Per-team producer of the node ring (one thread): stage pk goes to slot pk % S.
template <typename P, typename R, bool INTERP>
struct ResProducer {
  unsigned char* ring;
  unsigned long long *full, *empty;
  ResMeta* meta;
  int* pst;  // 0: sub, 1: base, 2: end, 3: tile, 4: pk
  __device__ __forceinline__ void load_sub(const int4* subs, int s, int nsubs) {
    pst[0] = s;
    if (s < nsubs) {
      const int4 sp = subs[s];
      pst[1] = sp.y;
      pst[2] = sp.y + sp.z;
      pst[3] = sp.x;
    }
  }
  template <typename F>
  __device__ __forceinline__ void produce(const R* psi, const unsigned* rrec, const void* xarr,
                                          const int4* subs, int nsubs, const Geom& g, int slot_id,
                                          int nteams, F&& on_new_sub) {
    constexpr int S = P::S, NB = P::NB;
    const int pk = pst[4];
    const int slot = pk % S;
    if (pk >= S) mbar_wait(empty + slot, ((pk / S) - 1) & 1);
    ResMeta* mt = meta + slot;
    pst[4] = pk + 1;
    if (pst[0] >= nsubs) {
      mt->nb = -1;
      mbar_arrive(full + slot);
      return;
    }
    const int pbase = pst[1], pend = pst[2];
    const int nb = min(NB, pend - pbase);
    const int off = pbase & 3;
    const int rcnt = (nb + off + 3) & ~3;
    mt->tile = pst[3];
    mt->nb = nb;
    mt->last = pbase + nb >= pend;
    mt->off = off;
    unsigned char* st = ring + slot * P::SB;
    const unsigned wb = (unsigned)(sizeof(R) * RES_PR) * nb, rb = 4u * rcnt;
    unsigned xb;
    const unsigned char* xsrc;
    if constexpr (INTERP) {
      xb = rb;
      xsrc = reinterpret_cast<const unsigned char*>(reinterpret_cast<const int*>(xarr) + (pbase - off));
    } else {
      constexpr int FA = P::FA;
      const int foff = pbase & (FA - 1);
      xb = (unsigned)P::ELEM * ((nb + foff + FA - 1) & ~(FA - 1));
      xsrc = reinterpret_cast<const unsigned char*>(xarr) + (size_t)P::ELEM * (pbase - foff);
    }
    mbar_expect_tx(full + slot, wb + rb + xb);
    bulk_g2s(st, psi + (int64_t)pbase * RES_PR, wb, full + slot);
    bulk_g2s(st + P::W_BYTES, rrec + (pbase - off), rb, full + slot);
    bulk_g2s(st + P::W_BYTES + P::R_BYTES, xsrc, xb, full + slot);
    if (pbase + nb < pend) {
      pst[1] = pbase + nb;
    } else {
      load_sub(subs, res_next_sub(g, slot_id, pst[0], nteams), nsubs);
      if (pst[0] < nsubs) on_new_sub(pst[1], pst[2] - pst[1], pst[3]);
    }
  }
};

// ------------------------------------------------------------------ B^H
// One node's operands for this lane, loaded one node ahead of its FMAs: the
// record, the lane's two leading-dim factors, the sample and the 2m last-dim
// factors (a team has two warps per SM sub-partition at most, so the load
// latency has to be covered inside the warp).
template <typename R>
struct ResNode {
  unsigned r;
  R wa, wb;
  cplx_t<R> f;
  R w2[RES_W];
};

#define NFFTK_RES_SPREAD_CASE(k)                          \
  case k:                                                 \
    _Pragma("unroll") for (int t = 0; t < RES_W; ++t) {   \
      accr[k + t] = fma(vr, w2[u][t], accr[k + t]);       \
      acci[k + t] = fma(vi, w2[u][t], acci[k + t]);       \
    }                                                     \
    break;

template <typename R, int NT, int NB, int S>
__global__ void __launch_bounds__(NT * 64, 1)
k_spread_res(cplx_t<R>* __restrict__ grid, const cplx_t<R>* __restrict__ fsorted,
             const R* __restrict__ psi, const unsigned* __restrict__ rrec,
             const int4* __restrict__ subs, int nsubs, Geom g) {
  using C = cplx_t<R>;
  using P = ResCfg<R, NT, NB, S, false>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int team = threadIdx.x >> 6, tt = threadIdx.x & 63, lane = threadIdx.x & 31;
  const int ra = tt >> 3, rb = tt & 7;
  unsigned char* tb = smem + team * P::TEAM_BYTES;
  C* halo = reinterpret_cast<C*>(tb);
  ResProducer<P, R, false> pr;
  pr.ring = tb + P::HALO;
  pr.full = reinterpret_cast<unsigned long long*>(pr.ring + S * P::SB);
  pr.empty = pr.full + S;
  pr.meta = reinterpret_cast<ResMeta*>(pr.empty + S + 2);
  pr.pst = reinterpret_cast<int*>(pr.meta + S);
  const int nteams = (int)gridDim.x * NT;
  // the next subproblem's node data is pulled into L2 when the producer draws it
  auto prefetch = [&](int base, int cnt, int) {
    l2_prefetch(psi + (int64_t)base * RES_PR, (unsigned)(sizeof(R) * RES_PR) * (unsigned)cnt);
    l2_prefetch(fsorted + (base & ~1), (unsigned)sizeof(C) * (unsigned)((cnt + 2) & ~1));
    l2_prefetch(rrec + (base & ~3), 4u * (unsigned)((cnt + 6) & ~3));
  };
  if (tt == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(pr.full + i, 1);
      mbar_init(pr.empty + i, 2);
    }
    pr.pst[4] = 0;
    pr.load_sub(subs, (int)blockIdx.x * NT + team, nsubs);
  }
  // the ring starts zeroed: the node loop reads whole groups of four, and a
  // batch's unused entries must hold finite factors (they are multiplied by 0)
  for (int i = tt; i < (int)(S * P::SB / 16); i += 64) reinterpret_cast<int4*>(pr.ring)[i] = make_int4(0, 0, 0, 0);
  fence_proxy_async_smem();
  team_sync(team);
  if (tt == 0)
    for (int i = 0; i < S; ++i) pr.produce(psi, rrec, fsorted, subs, nsubs, g, SCHED_SPREAD3, nteams, prefetch);

  R accr[RES_H], acci[RES_H];
#pragma unroll
  for (int c = 0; c < RES_H; ++c) accr[c] = acci[c] = 0;
  unsigned touched = 0;  // images of this lane written to the shared halo
  int cia = 0, cib = 0;  // image in registers: row (ra + 8 cia, rb + 8 cib)
  bool written = false;  // the image in registers has been entered by a node of this subproblem
  auto row_of = [&](int ia, int ib) { return halo + ((ra + 8 * ia) * RES_H + rb + 8 * ib) * RES_H; };
  auto store_row = [&]() {
    // the lane's previous bulk reductions have finished reading its rows
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    C* rw = row_of(cia, cib);
#pragma unroll
    for (int c = 0; c < RES_H; ++c) {
      C v;
      v.x = accr[c];
      v.y = acci[c];
      rw[c] = v;
    }
    touched |= 1u << (cia * 2 + cib);
  };
  int k = 0;
  for (;;) {  // subproblems of this team
    int tile = -1;
    unsigned cur_key = ~0u;  // no record has this key: the first node of a subproblem always takes the run path
    for (;; ++k) {  // batches of the subproblem
      const int slot = k % S;
      // refill the slot consumed one batch ago (both warps are past it)
      if (tt == 0 && k > 0) pr.produce(psi, rrec, fsorted, subs, nsubs, g, SCHED_SPREAD3, nteams, prefetch);
      mbar_wait(pr.full + slot, (k / S) & 1);
      const ResMeta mt = pr.meta[slot];
      if (mt.nb < 0) break;
      tile = mt.tile;
      const unsigned char* st = pr.ring + slot * P::SB;
      const R* pw = reinterpret_cast<const R*>(st);
      const unsigned* rs = reinterpret_cast<const unsigned*>(st + P::W_BYTES) + mt.off;
      const C* pf = reinterpret_cast<const C*>(st + P::W_BYTES + P::R_BYTES) + (P::FA > 1 ? (mt.off & (P::FA - 1)) : 0);
      // four nodes at a time: all their operands are requested before the
      // first FMA (a team has at most two warps per SM sub-partition, so the
      // shared-memory latency has to be covered inside the warp)
      for (int j0 = 0; j0 < mt.nb; j0 += 4) {
        unsigned r[4];
        R wa[4], wb[4], w2[4][RES_W];
        C f[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int jj = j0 + u;
          // past the batch: a record without RES_REGULAR (factor product zeroed below)
          r[u] = jj < mt.nb ? rs[jj] : 0u;
          const R* w = pw + jj * RES_PR;
          wa[u] = w[RES_W + ((ra - (int)r[u]) & 7)];
          wb[u] = w[2 * RES_W + ((rb - (int)(r[u] >> 3)) & 7)];
          f[u] = pf[jj];
          load8<R>(w, w2[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          R s = wa[u] * wb[u];
          // one test per node: a new (h0, h1) run or a wide node (its key
          // never equals a regular node's)
          if ((r[u] & RES_KEY) != cur_key) {
            if (!(r[u] & RES_REGULAR)) {
              s = 0;  // 2m+1 wide stencil: k_wide_nodes spreads it
            } else {
              cur_key = r[u] & RES_KEY;
              const int nia = ra < (int)(r[u] & 7), nib = rb < (int)((r[u] >> 3) & 7);
              if (nia != cia || nib != cib) {
                if (written) store_row();
                const C* rw = row_of(nia, nib);
                if (touched & (1u << (nia * 2 + nib))) {
#pragma unroll
                  for (int c = 0; c < RES_H; ++c) {
                    const C v = rw[c];
                    accr[c] = v.x;
                    acci[c] = v.y;
                  }
                } else {
#pragma unroll
                  for (int c = 0; c < RES_H; ++c) accr[c] = acci[c] = 0;
                }
                cia = nia;
                cib = nib;
              }
              written = true;
            }
          }
          const R vr = f[u].x * s, vi = f[u].y * s;
          switch ((r[u] >> 6) & 7) {
            NFFTK_RES_SPREAD_CASE(0) NFFTK_RES_SPREAD_CASE(1) NFFTK_RES_SPREAD_CASE(2) NFFTK_RES_SPREAD_CASE(3)
            NFFTK_RES_SPREAD_CASE(4) NFFTK_RES_SPREAD_CASE(5) NFFTK_RES_SPREAD_CASE(6) NFFTK_RES_SPREAD_CASE(7)
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(pr.empty + slot);
      if (mt.last) {
        ++k;
        break;
      }
    }
    if (tile < 0) break;  // end of work
    // subproblem done: every lane reduces the rows it wrote into the dense
    // grid (halo cell (a, b, c) = slot tile * 8 - (m - 1) + (a, b, c), wrapped)
    if (written) store_row();
#pragma unroll
    for (int c = 0; c < RES_H; ++c) accr[c] = acci[c] = 0;
    written = false;
    if (touched) {
      fence_proxy_async_smem();
      int tc[3];
      tile_of<3>(g, tile, tc);
      const int c0 = tc[2] * 8 - (g.m - 1);
#pragma unroll
      for (int img = 0; img < 4; ++img) {
        if (!(touched & (1u << img))) continue;
        const int a = ra + 8 * (img >> 1), b = rb + 8 * (img & 1);
        int ad = tc[0] * 8 - (g.m - 1) + a, bd = tc[1] * 8 - (g.m - 1) + b;
        ad += ad < 0 ? g.n[0] : (ad >= g.n[0] ? -g.n[0] : 0);
        bd += bd < 0 ? g.n[1] : (bd >= g.n[1] ? -g.n[1] : 0);
        bulk_red_row_wrapped<R>(grid, ((int64_t)ad * g.n[1] + bd) * g.n[2], c0, g.n[2],
                                halo + (a * RES_H + b) * RES_H, RES_H);
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::);
      touched = 0;
    }
  }
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
  team_sync(team);
  if (tt == 0) res_sched_done(g, SCHED_SPREAD3, nteams);
}

// -------------------------------------------------------------------- B
#define NFFTK_RES_INTERP_CASE(k)                           \
  case k:                                                  \
    _Pragma("unroll") for (int t = 0; t < RES_W; t += 2) { \
      p0r = fma(rowr[k + t], w2[u][t], p0r);               \
      p0i = fma(rowi[k + t], w2[u][t], p0i);               \
      p1r = fma(rowr[k + t + 1], w2[u][t + 1], p1r);       \
      p1i = fma(rowi[k + t + 1], w2[u][t + 1], p1i);       \
    }                                                      \
    break;

template <typename R, int NT, int NB, int S>
__global__ void __launch_bounds__(NT * 64, 1)
k_interp_res(const __grid_constant__ CUtensorMap tmap, cplx_t<R>* __restrict__ fout,
             const R* __restrict__ psi, const unsigned* __restrict__ rrec,
             const int* __restrict__ perm, const int4* __restrict__ subs, int nsubs, Geom g) {
  using C = cplx_t<R>;
  using P = ResCfg<R, NT, NB, S, true>;
  static_assert(NB % 4 == 0 && NB <= 32, "nodes are reduced four at a time, one combine lane per node");
  extern __shared__ __align__(128) unsigned char smem[];
  const int team = threadIdx.x >> 6, tt = threadIdx.x & 63, lane = threadIdx.x & 31, wt = tt >> 5;
  const int ra = tt >> 3, rb = tt & 7;
  unsigned char* tb = smem + team * P::TEAM_BYTES;
  const C* halo = reinterpret_cast<const C*>(tb);
  ResProducer<P, R, true> pr;
  pr.ring = tb + P::HALO;
  pr.full = reinterpret_cast<unsigned long long*>(pr.ring + S * P::SB);
  pr.empty = pr.full + S;
  unsigned long long* hfull = pr.empty + S;
  unsigned long long* hempty = hfull + 1;
  pr.meta = reinterpret_cast<ResMeta*>(pr.empty + S + 2);
  pr.pst = reinterpret_cast<int*>(pr.meta + S);
  // per slot: the two warps' sums of the batch's nodes (combined by warp 0
  // when both are past the batch, before the slot is refilled)
  C* part = reinterpret_cast<C*>(pr.ring + S * P::SB + P::CTL);
  const int nteams = (int)gridDim.x * NT;
  constexpr int SCALE = (int)sizeof(C) / 8;
  auto box_of = [&](int tile, int* c) {
    int tc[3];
    tile_of<3>(g, tile, tc);
    // halo cell 0 = slot tile * 8 - (m - 1) = padded index tile * 8 + 1
    c[0] = (tc[2] * 8 + 1) * SCALE;
    c[1] = tc[1] * 8 + 1;
    c[2] = tc[0] * 8 + 1;
  };
  // the next subproblem's halo and node data are pulled into L2 as soon as the producer draws it
  auto prefetch = [&](int base, int cnt, int tile) {
    int c[3];
    box_of(tile, c);
    tma_prefetch_box3(&tmap, c);
    l2_prefetch(psi + (int64_t)base * RES_PR, (unsigned)(sizeof(R) * RES_PR) * (unsigned)cnt);
    l2_prefetch(perm + (base & ~3), 4u * (unsigned)((cnt + 6) & ~3));
    l2_prefetch(rrec + (base & ~3), 4u * (unsigned)((cnt + 6) & ~3));
  };
  if (tt == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(pr.full + i, 1);
      mbar_init(pr.empty + i, 2);
    }
    mbar_init(hfull, 1);
    mbar_init(hempty, 2);
    pr.pst[4] = 0;
    pr.load_sub(subs, (int)blockIdx.x * NT + team, nsubs);
    for (int i = 0; i < S; ++i) pr.produce(psi, rrec, perm, subs, nsubs, g, SCHED_INTERP, nteams, prefetch);
  }
  team_sync(team);

  R rowr[RES_H], rowi[RES_H];
  unsigned cur_key = ~0u;  // no record has this key
  int cia = -1, cib = -1;
  // warp 0: f[perm] = both warps' sums of batch kk (its slot is about to be refilled)
  auto combine = [&](int kk) {
    const int slot = kk % S;
    if (lane == 0) mbar_wait(pr.empty + slot, (kk / S) & 1);
    __syncwarp();
    const ResMeta mt = pr.meta[slot];
    const unsigned char* st = pr.ring + slot * P::SB;
    const unsigned* rs = reinterpret_cast<const unsigned*>(st + P::W_BYTES) + mt.off;
    const int* pv = reinterpret_cast<const int*>(st + P::W_BYTES + P::R_BYTES) + mt.off;
    if (lane < mt.nb && (rs[lane] & RES_REGULAR)) {
      const C a = part[(slot * 2) * NB + lane], b = part[(slot * 2 + 1) * NB + lane];
      C v;
      v.x = a.x + b.x;
      v.y = a.y + b.y;
      fout[pv[lane]] = v;
    }
    __syncwarp();
  };
  int k = 0;
  for (int it = 0;; ++it) {  // subproblems of this team
    if (wt == 0 && k > 0) {
      combine(k - 1);
      if (lane == 0) pr.produce(psi, rrec, perm, subs, nsubs, g, SCHED_INTERP, nteams, prefetch);
    }
    mbar_wait(pr.full + k % S, (k / S) & 1);
    const ResMeta m0 = pr.meta[k % S];
    if (m0.nb < 0) break;
    if (tt == 0) {
      if (it > 0) mbar_wait(hempty, (it - 1) & 1);  // both warps are done with the previous halo
      int c[3];
      box_of(m0.tile, c);
      mbar_expect_tx(hfull, (unsigned)(RES_H * RES_H * P::ROW));
      tma_load_box<3>(tb, &tmap, c, hfull);
    }
    mbar_wait(hfull, it & 1);
    cur_key = ~0u;
    cia = cib = -1;
    for (bool first = true;; ++k, first = false) {  // batches of the subproblem
      const int slot = k % S;
      if (!first && wt == 0) {
        combine(k - 1);
        if (lane == 0) pr.produce(psi, rrec, perm, subs, nsubs, g, SCHED_INTERP, nteams, prefetch);
      }
      mbar_wait(pr.full + slot, (k / S) & 1);
      const ResMeta mt = pr.meta[slot];
      const unsigned char* st = pr.ring + slot * P::SB;
      const R* pw = reinterpret_cast<const R*>(st);
      const unsigned* rs = reinterpret_cast<const unsigned*>(st + P::W_BYTES) + mt.off;
      for (int j = 0; j < mt.nb; j += 4) {
        // four nodes: all their operands are requested up front, then one
        // transposing reduction -- lanes keep half of the values at each of
        // the first two exchanges (24 shuffles for four nodes instead of 80)
        unsigned r[4];
        R wa[4], wb[4], w2[4][RES_W];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int jj = min(j + u, mt.nb - 1);
          r[u] = rs[jj];
          const R* w = pw + jj * RES_PR;
          wa[u] = w[RES_W + ((ra - (int)r[u]) & 7)];
          wb[u] = w[2 * RES_W + ((rb - (int)(r[u] >> 3)) & 7)];
          load8<R>(w, w2[u]);
        }
        R vr[4], vi[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          R s = wa[u] * wb[u];
          if ((r[u] & RES_KEY) != cur_key) {  // a new (h0, h1) run, or a wide node
            if (!(r[u] & RES_REGULAR)) {
              s = 0;  // 2m+1 wide stencil: k_wide_nodes
            } else {
              cur_key = r[u] & RES_KEY;
              const int nia = ra < (int)(r[u] & 7), nib = rb < (int)((r[u] >> 3) & 7);
              if (nia != cia || nib != cib) {
                const C* rw = halo + ((ra + 8 * nia) * RES_H + rb + 8 * nib) * RES_H;
#pragma unroll
                for (int c = 0; c < RES_H; ++c) {
                  const C v = rw[c];
                  rowr[c] = v.x;
                  rowi[c] = v.y;
                }
                cia = nia;
                cib = nib;
              }
            }
          }
          R p0r = 0, p0i = 0, p1r = 0, p1i = 0;
          switch ((r[u] >> 6) & 7) {
            NFFTK_RES_INTERP_CASE(0) NFFTK_RES_INTERP_CASE(1) NFFTK_RES_INTERP_CASE(2) NFFTK_RES_INTERP_CASE(3)
            NFFTK_RES_INTERP_CASE(4) NFFTK_RES_INTERP_CASE(5) NFFTK_RES_INTERP_CASE(6) NFFTK_RES_INTERP_CASE(7)
          }
          vr[u] = (p0r + p1r) * s;
          vi[u] = (p0i + p1i) * s;
        }
        const bool hi16 = lane & 16, hi8 = lane & 8;
        // xor 16: lanes 0-15 keep nodes 0, 1; lanes 16-31 keep nodes 2, 3
        R kr0 = hi16 ? vr[2] : vr[0], ki0 = hi16 ? vi[2] : vi[0], kr1 = hi16 ? vr[3] : vr[1],
          ki1 = hi16 ? vi[3] : vi[1];
        kr0 += __shfl_xor_sync(0xffffffffu, hi16 ? vr[0] : vr[2], 16);
        ki0 += __shfl_xor_sync(0xffffffffu, hi16 ? vi[0] : vi[2], 16);
        kr1 += __shfl_xor_sync(0xffffffffu, hi16 ? vr[1] : vr[3], 16);
        ki1 += __shfl_xor_sync(0xffffffffu, hi16 ? vi[1] : vi[3], 16);
        // xor 8: keep one node: n = 2 * bit4 + bit3
        R sr = hi8 ? kr1 : kr0, si = hi8 ? ki1 : ki0;
        sr += __shfl_xor_sync(0xffffffffu, hi8 ? kr0 : kr1, 8);
        si += __shfl_xor_sync(0xffffffffu, hi8 ? ki0 : ki1, 8);
#pragma unroll
        for (int o = 4; o; o >>= 1) {
          sr += __shfl_xor_sync(0xffffffffu, sr, o);
          si += __shfl_xor_sync(0xffffffffu, si, o);
        }
        if ((lane & 7) == 0) {
          C v;
          v.x = sr;
          v.y = si;
          part[(slot * 2 + wt) * NB + j + (lane >> 3)] = v;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(pr.empty + slot);
      if (mt.last) {
        ++k;
        break;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(hempty);
  }
  team_sync(team);
  if (tt == 0) res_sched_done(g, SCHED_INTERP, nteams);
}


// ------------------------------------------------ nodes with 2m+1 wide stencils
// One warp per such node (rare: n x an exact integer in some dim): window
// factors evaluated directly (kernels.py:42-53), the stencil walked by the
// lanes; spread with atomics into the dense grid, interp with a warp sum.
template <typename R, bool SPREAD>
__global__ void __launch_bounds__(256)
k_wide_nodes(cplx_t<R>* __restrict__ grid, cplx_t<R>* __restrict__ f, const unsigned* __restrict__ rrec,
             const double* __restrict__ xs, const int* __restrict__ perm, Geom g) {
  // SPREAD: grid is the dense n-grid; interp: the ghost-padded copy (slot s at s + m)
  using C = cplx_t<R>;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int K = 2 * g.m + 1;
  for (int64_t base = w0 * 32; base < g.M; base += nw * 32) {
    const int64_t i = base + lane;
    unsigned todo = __ballot_sync(~0u, i < g.M && !(rrec[i] & RES_REGULAR));
    while (todo) {
      const int64_t j = base + __ffs(todo) - 1;
      todo &= todo - 1;
      // lanes 0 .. 3K-1 evaluate the (dim, offset) factors once
      int64_t lo[3];
      int wd[3];
#pragma unroll
      for (int dim = 0; dim < 3; ++dim) {
        const Stencil st = stencil(xs[dim * g.M + j], g.nd[dim], g.md);
        lo[dim] = st.lo;
        wd[dim] = st.width;
      }
      double fac = 0.0;
      if (lane < 3 * K) {
        const int dim = lane / K, t = lane - dim * K;
        if (t < wd[dim]) fac = dim_factor(g, dim, xs[dim * g.M + j], lo[dim] + t) * g.wscale[dim];
      }
      C fj = C{0, 0};
      if (SPREAD) fj = f[j];
      double sr = 0, si = 0;
      const int cells = wd[0] * wd[1] * wd[2];
      for (int q0 = 0; q0 < cells; q0 += 32) {
        const int q = q0 + lane;
        const bool on = q < cells;
        const int qq = on ? q : 0;
        const int t2 = qq % wd[2], t1 = (qq / wd[2]) % wd[1], t0 = qq / (wd[2] * wd[1]);
        const double f0 = __shfl_sync(~0u, fac, t0), f1 = __shfl_sync(~0u, fac, K + t1),
                     f2 = __shfl_sync(~0u, fac, 2 * K + t2);
        if (!on) continue;
        const double wgt = f0 * f1 * f2;
        const int64_t s0 = floor_mod(lo[0] + t0, g.n[0]), s1 = floor_mod(lo[1] + t1, g.n[1]),
                      s2 = floor_mod(lo[2] + t2, g.n[2]);
        const int64_t idx = SPREAD ? (s0 * g.n[1] + s1) * g.n[2] + s2
                                   : ((s0 + g.m) * g.np[1] + s1 + g.m) * g.np[2] + s2 + g.m;
        if (SPREAD) {
          atomicAdd(&grid[idx].x, (R)(fj.x * wgt));
          atomicAdd(&grid[idx].y, (R)(fj.y * wgt));
        } else {
          const C v = grid[idx];
          sr += (double)v.x * wgt;
          si += (double)v.y * wgt;
        }
      }
      if (!SPREAD) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          sr += __shfl_xor_sync(~0u, sr, o);
          si += __shfl_xor_sync(~0u, si, o);
        }
        if (lane == 0) {
          C v;
          v.x = (R)sr;
          v.y = (R)si;
          f[perm[j]] = v;
        }
      }
    }
  }
}

// ================================================================ launchers
bool res_geometry(const Geom& g, bool single) {
  if (getenv("NFFTK_NO_RES") || getenv("NFFTK_NO_PIPE") || getenv("NFFTK_NO_DENSE_FLUSH")) return false;
  if (single) return false;
  if (g.d != 3 || g.m != RES_M) return false;
  for (int i = 0; i < 3; ++i)
    if (g.T[i] != 8 || g.n[i] < 8 + 2 * RES_M + 1) return false;
  return true;
}

bool res_ok(const Geom& g) {
  return g.res && g.mode == MODE_TENSOR && g.psi && g.rrec && g.psi_pad == 3 && g.dense_flush;
}

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    NFFTK_CUDA(cudaGetDevice(&dev));
    NFFTK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

static Geom res_sched_geom(const Geom& g, int nsubs, int nteams) {
  Geom q = g;
  if ((int64_t)nsubs < 4LL * nteams) q.sched = nullptr;
  return q;
}

template <int NT, int NB, int S>
static void spread_res_go(void* grid, const void* fs, const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  using P = ResCfg<double, NT, NB, S, false>;
  static_assert(P::SMEM <= 227 * 1024, "residue spread: shared memory");
  auto kern = k_spread_res<double, NT, NB, S>;
  NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
  const int grid_x = std::max(1, std::min((nsubs + NT - 1) / NT, sm_count()));
  kern<<<grid_x, P::THREADS, P::SMEM, s>>>((double2*)grid, (const double2*)fs, g.psi, g.rrec, subs, nsubs,
                                          res_sched_geom(g, nsubs, grid_x * NT));
  count_launch();
}

template <int NT, int NB, int S>
static void interp_res_go(const CUtensorMap* tm, void* f, const int* perm, const int4* subs, int nsubs,
                          const Geom& g, cudaStream_t s) {
  using P = ResCfg<double, NT, NB, S, true>;
  static_assert(P::SMEM <= 227 * 1024, "residue interp: shared memory");
  auto kern = k_interp_res<double, NT, NB, S>;
  NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
  const int grid_x = std::max(1, std::min((nsubs + NT - 1) / NT, sm_count()));
  kern<<<grid_x, P::THREADS, P::SMEM, s>>>(*tm, (double2*)f, g.psi, g.rrec, perm, subs, nsubs,
                                          res_sched_geom(g, nsubs, grid_x * NT));
  count_launch();
}

static int res_teams() {
  static int nt = 0;
  if (!nt) {
    const char* e = getenv("NFFTK_RES_TEAMS");
    nt = e ? atoi(e) : 4;
    if (nt != 3 && nt != 4) nt = 4;
  }
  return nt;
}

// B^H into the dense grid (zeroed by the caller): regular nodes by the
// residue kernel, wide ones (g.nwide of them) by k_wide_nodes.
void launch_spread_res(void* grid, const void* fs, const double* xs, const int4* subs, int nsubs,
                       const Geom& g, cudaStream_t s) {
  if (res_teams() == 3) spread_res_go<3, 16, 6>(grid, fs, subs, nsubs, g, s);
  else spread_res_go<4, 4, 4>(grid, fs, subs, nsubs, g, s);
  if (g.nwide > 0) {
    Geom q = g;
    q.mode = MODE_DIRECT;
    k_wide_nodes<double, true><<<sm_count() * 4, 256, 0, s>>>((double2*)grid, (double2*)fs, g.rrec, xs, nullptr, q);
    count_launch();
  }
}

// B from the ghost-padded grid gp (tensor map tm: 15^3 boxes); f is zeroed first (the two
// warps of a team add their halves of a sample).
void launch_interp_res(const void* tm, const void* gp, void* f, const double* xs, const int* perm,
                       const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  NFFTK_CUDA(cudaMemsetAsync(f, 0, sizeof(double2) * (size_t)g.M, s));
  if (res_teams() == 3) interp_res_go<3, 16, 6>((const CUtensorMap*)tm, f, perm, subs, nsubs, g, s);
  else interp_res_go<4, 4, 4>((const CUtensorMap*)tm, f, perm, subs, nsubs, g, s);
  if (g.nwide > 0) {
    Geom q = g;
    q.mode = MODE_DIRECT;
    k_wide_nodes<double, false><<<sm_count() * 4, 256, 0, s>>>((double2*)gp, (double2*)f, g.rrec, xs, perm, q);
    count_launch();
  }
}

}  // namespace nfftk
