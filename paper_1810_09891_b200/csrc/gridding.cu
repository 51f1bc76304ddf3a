// Gridding kernels of the nfftk hot path (sm_100a):
//   B   (interp) : f_j = sum_l g[l mod n] prod_i psi_i(x_ji - l_i / n_i)
//   B^H (spread) : g[l mod n] += f_j prod_i psi_i(x_ji - l_i / n_i)
// Reference: kernels.py:122-197 (gather_{1,2,3}d), :209-401 (spread_*).
//
// Both work on tile subproblems produced by the device sort (kernels.cu):
// one CTA per (tile, <= maxsub nodes).  The tile's (T + 2m + 1)^d halo lives
// in shared memory.  The grid they read / write is the ghost-padded copy
// (plan.cu: pad / fold kernels keep the periodic images), so every halo is
// ONE contiguous box:
//   * interp loads it with a single TMA tensor copy (cp.async.bulk.tensor,
//     completion on an mbarrier);
//   * spread flushes it with TMA bulk fp64 (fp32) reductions into L2
//     (cp.reduce.async.bulk .add), one per halo row -- no per-cell atomics.
// Node batches (coordinates, samples, PRE_PSI factors) arrive by cp.async into
// a double buffer while the previous batch is processed.
//
// Halo rows along the last dimension have stride HS (= H for complex128,
// which is odd and keeps lane-strided 128-bit accesses bank-conflict free).
// Kernels are templated on the cutoff MM (1..8; 0 = runtime m) so the 2m-wide
// stencil loops unroll; nodes whose stencil is 2m+1 wide in some dimension
// (n x an exact integer, or fp rounding at the edges -- common.cuh
// ``stencil``) take a generic path with runtime widths.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "async.cuh"
#include "common.cuh"
#include "kernels.h"

namespace nfftk {


// ----------------------------------------------------------- node batches
// coordinates [D][NB], window factors [NB][D*K] (PRE_PSI rows copied, or
// computed), stencil data hw[NB][2D+1] = {h_0..h_{D-1}, W_0..W_{D-1}, fast},
// interp output index pb[NB], spread sorted samples fv[NB].
template <typename C, int D>
struct Batch {
  double* x;
  double* w;
  int* hw;
  int* pb;
  C* fv;
};

__host__ __device__ inline size_t batch_bytes_of(int d, int nb, int K, int elem) {
  auto al = [](size_t v) { return (v + 15) & ~(size_t)15; };
  return al(sizeof(double) * d * nb) + al(sizeof(double) * nb * psi_row(d, K)) +
         al(sizeof(int) * nb * (2 * d + 2)) + al(sizeof(int) * nb) + al((size_t)elem * nb);
}

template <typename C, int D>
__device__ __forceinline__ Batch<C, D> batch_at(unsigned char* p, int nb, int K) {
  Batch<C, D> b;
  b.x = reinterpret_cast<double*>(p);
  p += a16(sizeof(double) * D * nb);
  b.w = reinterpret_cast<double*>(p);
  p += a16(sizeof(double) * nb * psi_row(D, K));
  b.hw = reinterpret_cast<int*>(p);
  p += a16(sizeof(int) * nb * (2 * D + 2));
  b.pb = reinterpret_cast<int*>(p);
  p += a16(sizeof(int) * nb);
  b.fv = reinterpret_cast<C*>(p);
  return b;
}

template <typename C, int D>
__device__ __forceinline__ void issue_batch(const Geom& g, const double* __restrict__ xs,
                                            const int* __restrict__ perm, const C* __restrict__ fs,
                                            int base, int nb, int NB, const Batch<C, D>& b) {
  const int K = 2 * g.m + 1, per = psi_row(D, K);
  for (int q = threadIdx.x; q < D * nb; q += blockDim.x) {
    int dim = q / nb, j = q - dim * nb;
    cp_async8(b.x + dim * NB + j, xs + dim * g.M + base + j);
  }
  if (perm)
    for (int j = threadIdx.x; j < nb; j += blockDim.x) cp_async4(b.pb + j, perm + base + j);
  if (fs)
    for (int j = threadIdx.x; j < nb; j += blockDim.x) cp_async_cell(b.fv + j, fs + base + j);
  if (g.mode == MODE_TENSOR) {
    const double* src = g.psi + (int64_t)base * per;
    for (int q = threadIdx.x; q < nb * per; q += blockDim.x) cp_async8(b.w + q, src + q);
  }
}

// Stencils in halo coordinates, h = (cell slot - tile start) + m - (cell - lo)
// in [0, T + m + 1]; the fast flag (width 2m in every dim); (DIRECT / LUT)
// window factors -- kernels.py:42-53 for a whole batch.
template <typename C, int D>
__device__ __forceinline__ void finish_batch(const Geom& g, const int* tc, int nb, int NB, int ua,
                                             const Batch<C, D>& b) {
  const int K = 2 * g.m + 1, per = psi_row(D, K);
  for (int j = threadIdx.x; j < nb; j += blockDim.x) {
    bool fast = true;
    int* q = b.hw + j * (2 * D + 2);
#pragma unroll
    for (int dim = 0; dim < D; ++dim) {
      Stencil st = stencil(b.x[dim * NB + j], g.nd[dim], g.md);
      int slot = (int)floor_mod(st.cell, g.n[dim]);
      q[dim] = slot - tc[dim] * g.T[dim] + g.m - (int)(st.cell - st.lo);
      q[D + dim] = st.width;
      fast = fast && st.width == 2 * g.m;
    }
    q[2 * D] = fast;
    q[2 * D + 1] = q[0] % ua;
  }
  if (g.mode != MODE_TENSOR) {
    for (int q = threadIdx.x; q < nb * per; q += blockDim.x) {
      int j = q / per, r = q - j * per, dim = r / K, t = r - dim * K;
      if (dim >= D) {  // row padding
        b.w[q] = 0.0;
        continue;
      }
      double x = b.x[dim * NB + j];
      Stencil st = stencil(x, g.nd[dim], g.md);
      b.w[q] = t < st.width ? dim_factor(g, dim, x, st.lo + t) * g.wscale[dim] : 0.0;
    }
  }
}

// Lanes per node in the interp: enough work per lane to amortise the
// per-node fixed cost; a power of two so the team reduction stays in-warp.
template <int D, int MM>
struct InterpTeam {
  static constexpr int WF = 2 * (MM > 0 ? MM : 1);
  static constexpr int P = D == 3 ? WF * WF : (D == 2 ? 2 * WF : WF);
  static constexpr int value =
      MM > 0 ? (D == 3 ? (P >= 128 ? 16 : 8) : (D == 2 ? (P >= 24 ? 8 : 4) : 16)) : 32;
};

// ======================================================== B: interpolation
// One CTA per subproblem.  One TMA copy brings the halo box while the first
// node batch arrives by cp.async; the next batch is fetched while the current
// one is processed.  A team of TEAM lanes reduces one node: lanes split the
// leading stencil dims and run along the contiguous last dim with the factors
// in registers; a team shuffle reduction forms f_j.
// One node of the interpolation, this lane's share (lane tl of a TEAM):
// q = {h_0..h_{D-1}, W_0..W_{D-1}, fast}.  The factor of stencil offset t in
// leading dim 0 / 1 is w0[o0 + t] / w1[o1 + t] (o = 0 for stencil-indexed
// rows, the stencil start h for halo-indexed PRE_PSI rows); wl holds the
// last-dim factors.
template <typename R, int D, int MM, int TEAM, typename W>
__device__ __forceinline__ void interp_node(const cplx_t<R>* __restrict__ halo, int HS, int H1, int K,
                                            const int* q, const W* w0, const W* w1,
                                            const W* wl, int o0, int o1, int tl, R& are,
                                            R& aim, int sh = 0) {
  using C = cplx_t<R>;
  if (MM > 0 && q[2 * D]) {
    constexpr int WF = 2 * (MM > 0 ? MM : 1);
    if constexpr (D == 1) {
      for (int t0 = tl; t0 < WF; t0 += TEAM) {
        C v = halo[q[0] + t0];
        R ww = (R)wl[t0];
        are = fma(ww, v.x, are);
        aim = fma(ww, v.y, aim);
      }
    } else if constexpr (D == 2) {
      // lanes own whole stencil rows: a TEAM of consecutive halo rows hits
      // distinct shared-memory banks (odd row stride)
      R w1r[WF];
#pragma unroll
      for (int t = 0; t < WF; ++t) w1r[t] = (R)wl[t];
      if constexpr (WF == 12 && TEAM == 8 && sizeof(R) == 8) {
        // 12 rows on 8 lanes: rows 0..7 whole, then rows 8..11 split between
        // lane pairs.  With an odd row stride the 4 rows a phase-2 quarter
        // warp reads start in the bank-group set D = {0, 2, 5, 7} (+ shift);
        // the two halves read columns u and u + 4 -- D and D + 4 are
        // disjoint, so those loads are conflict-free -- then columns 8..9 /
        // 10..11.  20 instead of 24 wavefronts per node (half the lanes
        // idled through rows 8..11 before).
        {
          const C* row = halo + (q[0] + tl) * HS + q[1];
          R sre = 0, sim = 0;
#pragma unroll
          for (int t = 0; t < WF; ++t) {
            C v = row[t];
            sre = fma(w1r[t], v.x, sre);
            sim = fma(w1r[t], v.y, sim);
          }
          R f0 = (R)w0[o0 + tl];
          are = fma(f0, sre, are);
          aim = fma(f0, sim, aim);
        }
        const int j = tl & 3, h = tl >> 2;
        const C* row = halo + (q[0] + 8 + j) * HS + q[1];
        R sre = 0, sim = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          C v = row[u + 4 * h];
          const R w = h ? w1r[u + 4] : w1r[u];
          sre = fma(w, v.x, sre);
          sim = fma(w, v.y, sim);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          C v = row[8 + 2 * h + u];
          const R w = h ? w1r[10 + u] : w1r[8 + u];
          sre = fma(w, v.x, sre);
          sim = fma(w, v.y, sim);
        }
        R f0 = (R)w0[o0 + 8 + j];
        are = fma(f0, sre, are);
        aim = fma(f0, sim, aim);
      } else {
        for (int t0 = tl; t0 < WF; t0 += TEAM) {
          const C* row = halo + (q[0] + t0) * HS + q[1];
          R sre = 0, sim = 0;
#pragma unroll
          for (int t = 0; t < WF; ++t) {
            C v = row[t];
            sre = fma(w1r[t], v.x, sre);
            sim = fma(w1r[t], v.y, sim);
          }
          R f0 = (R)w0[o0 + t0];
          are = fma(f0, sre, are);
          aim = fma(f0, sim, aim);
        }
      }
    } else {
      R w2r[WF];
#pragma unroll
      for (int t = 0; t < WF; ++t) w2r[t] = (R)wl[t];
      const C* corner = halo + (q[0] * H1 + q[1]) * HS + q[2];
      if constexpr (TEAM == WF && sizeof(R) == 4) {
        // complex64, 8-lane teams: a half warp (one 8-byte shared-memory
        // wavefront) holds two teams, whose rows start an even number of
        // 4-byte words apart -- they collide in the banks whenever the two
        // nodes' last-dim starts have the same parity (half of the time: 1.5
        // wavefronts per load, ncu: 32% of the gather's wavefronts were
        // conflicts).  sh = 1 tells the odd team of such a pair to walk its
        // rows rotated by one cell (cells 1..7, then 0): the two footprints
        // interleave and every load is one wavefront.
        const R f1 = (R)w1[o1 + tl];
        R wa[WF - 1];
#pragma unroll
        for (int t = 0; t < WF - 1; ++t) wa[t] = sh ? w2r[t + 1] : w2r[t];
        const R wlast = sh ? w2r[0] : w2r[WF - 1];
        const int dl = sh ? 0 : WF - 1;
        const C* row = corner + tl * HS;
#pragma unroll 2
        for (int t0 = 0; t0 < WF; ++t0, row += H1 * HS) {
          const C* p1 = row + sh;
          R sre = 0, sim = 0;
#pragma unroll
          for (int t = 0; t < WF - 1; ++t) {
            C v = p1[t];
            sre = fma(wa[t], v.x, sre);
            sim = fma(wa[t], v.y, sim);
          }
          {
            C v = row[dl];
            sre = fma(wlast, v.x, sre);
            sim = fma(wlast, v.y, sim);
          }
          R w01 = (R)(w0[o0 + t0] * f1);
          are = fma(w01, sre, are);
          aim = fma(w01, sim, aim);
        }
      } else if constexpr (TEAM == WF) {
        // lane tl walks the WF rows (t0, tl), t0 = 0 .. WF-1: its dim-1
        // factor is fixed and the row pointer advances by one halo plane --
        // no per-row index arithmetic, one factor load less per row
        const R f1 = (R)w1[o1 + tl];
        const C* row = corner + tl * HS;
#pragma unroll 2
        for (int t0 = 0; t0 < WF; ++t0, row += H1 * HS) {
          R sre = 0, sim = 0;
#pragma unroll
          for (int t = 0; t < WF; ++t) {
            C v = row[t];
            sre = fma(w2r[t], v.x, sre);
            sim = fma(w2r[t], v.y, sim);
          }
          R w01 = (R)(w0[o0 + t0] * f1);
          are = fma(w01, sre, are);
          aim = fma(w01, sim, aim);
        }
      } else
#pragma unroll 2
      for (int p = tl; p < WF * WF; p += TEAM) {
        int t0 = p / WF, t1 = p - t0 * WF;
        const C* row = corner + (t0 * H1 + t1) * HS;
        R sre = 0, sim = 0;
#pragma unroll
        for (int t = 0; t < WF; ++t) {
          C v = row[t];
          sre = fma(w2r[t], v.x, sre);
          sim = fma(w2r[t], v.y, sim);
        }
        R w01 = (R)(w0[o0 + t0] * w1[o1 + t1]);
        are = fma(w01, sre, are);
        aim = fma(w01, sim, aim);
      }
    }
  } else {
    // generic widths (2m or 2m+1 per dim), runtime loops
    if constexpr (D == 1) {
      for (int t0 = tl; t0 < q[1]; t0 += TEAM) {
        C v = halo[q[0] + t0];
        R ww = (R)wl[t0];
        are = fma(ww, v.x, are);
        aim = fma(ww, v.y, aim);
      }
    } else {
      const int WL = q[2 * D - 1];
      const int P = D == 2 ? q[D] : q[D] * q[D + 1];
      const int W1 = D == 3 ? q[D + 1] : 1;
      for (int p = tl; p < P; p += TEAM) {
        int t0 = p / W1, t1 = p - t0 * W1;
        const C* row = D == 2 ? halo + (q[0] + t0) * HS + q[1]
                              : halo + ((q[0] + t0) * H1 + q[1] + t1) * HS + q[D - 1];
        R sre = 0, sim = 0;
        for (int t = 0; t < WL; ++t) {
          C v = row[t];
          sre = fma((R)wl[t], v.x, sre);
          sim = fma((R)wl[t], v.y, sim);
        }
        R wr = (R)(D == 2 ? w0[o0 + t0] : w0[o0 + t0] * w1[o1 + t1]);
        are = fma(wr, sre, are);
        aim = fma(wr, sim, aim);
      }
    }
  }
}

// Bank-conflict-free row schedule for the d = 3 c128 gather.  A TEAM lane
// walks whole stencil rows (t0, t1) of 2m cells; one LDS.128 of 32 lanes is
// served per quarter warp, so the 8 rows a quarter warp reads together must
// start in 8 different 16-byte bank groups.  Row (t0, t1) starts in group
// (alpha t0 + beta t1 + corner) mod 8 with alpha = H1 HS, beta = HS (the
// corner shift is common to the team).  The natural order p = tl + TEAM k
// wraps t1 at 2m and collides whenever 2m is not a multiple of 8 (m = 5, 6:
// ~23% extra wavefronts at m = 6); this schedule deals the rows out class by
// class instead.  Entries are t0 << 8 | t1, 0xffff = no row.
template <int WF, int TEAM, int H1, int HS>
struct RowSched {
  static constexpr int P = WF * WF;
  static constexpr int NIT = (P + TEAM - 1) / TEAM;
  unsigned short v[NIT * TEAM];
  constexpr RowSched() : v() {
    bool used[P] = {};
    const int alpha = (H1 * HS) % 8, beta = HS % 8;
    for (int slot = 0; slot < NIT * TEAM; slot += 8) {  // one quarter warp
      bool cls[8] = {};
      for (int l = 0; l < 8; ++l) {
        int pick = -1;
        // the unused row of a free class whose class has the most rows left
        int best = -1;
        for (int c = 0; c < 8; ++c) {
          if (cls[c]) continue;
          int left = 0, first = -1;
          for (int r = 0; r < P; ++r)
            if (!used[r] && (alpha * (r / WF) + beta * (r % WF)) % 8 == c) {
              ++left;
              if (first < 0) first = r;
            }
          if (left > best && first >= 0) {
            best = left;
            pick = first;
          }
        }
        if (pick < 0)  // every free class is empty: any unused row (conflict)
          for (int r = 0; r < P && pick < 0; ++r)
            if (!used[r]) pick = r;
        if (pick < 0) {
          v[slot + l] = 0xffff;
          continue;
        }
        used[pick] = true;
        cls[(alpha * (pick / WF) + beta * (pick % WF)) % 8] = true;
        v[slot + l] = (unsigned short)((pick / WF) << 8 | (pick % WF));
      }
    }
  }
};

template <int WF, int TEAM, int H1, int HS>
__constant__ RowSched<WF, TEAM, H1, HS> c_row_sched = RowSched<WF, TEAM, H1, HS>();

// One fast (width 2m in every dim) c128 node of the d = 3 gather on the
// schedule above; sch[] holds this lane's rows.
template <int MM, int TEAM, int H1, int HS>
__device__ __forceinline__ void interp_node3_sched(const double2* __restrict__ halo, const int* q,
                                                   const double* w0, const double* w1,
                                                   const double* wl, int o0, int o1,
                                                   const unsigned* sch, double& are, double& aim) {
  constexpr int WF = 2 * MM;
  constexpr int NIT = RowSched<WF, TEAM, H1, HS>::NIT;
  double w2r[WF];
#pragma unroll
  for (int t = 0; t < WF; ++t) w2r[t] = wl[t];
  const double2* corner = halo + (q[0] * H1 + q[1]) * HS + q[2];
  // fully unrolled: sch[] stays in registers (a partial unroll indexed it
  // from local memory: C3 interp 0.351 -> 0.343 ms, c64 0.217 -> 0.208)
#pragma unroll
  for (int k = 0; k < NIT; ++k) {
    const unsigned e = sch[k];
    if (e == 0xffffu) continue;
    const int t0 = e >> 8, t1 = e & 0xff;
    const double2* row = corner + (t0 * H1 + t1) * HS;
    double sre = 0, sim = 0;
#pragma unroll
    for (int t = 0; t < WF; ++t) {
      const double2 v = row[t];
      sre = fma(w2r[t], v.x, sre);
      sim = fma(w2r[t], v.y, sim);
    }
    const double w01 = w0[o0 + t0] * w1[o1 + t1];
    are = fma(w01, sre, are);
    aim = fma(w01, sim, aim);
  }
}

// One fast c64 node of the d = 3 gather.  c64 halo rows have an even stride
// (HS = H + 1 keeps TMA rows 16-byte), so whole-row lanes start in only half
// of the 8-byte bank pairs; here a TEAM of 16 is 8 row slots x 2 parities:
// the two lanes of a slot read the even / odd cells of one row, and the 8
// rows a half warp reads together come from RowSched over 16-byte units
// (HS / 2), so the 16 lanes hit 16 different bank pairs.
template <int MM, int H1, int HS>
__device__ __forceinline__ void interp_node3_half(const float2* __restrict__ halo, const int* q,
                                                  const float* w0, const float* w1,
                                                  const float* wl, int o0, int o1, int par,
                                                  const unsigned* sch, float& are, float& aim) {
  constexpr int WF = 2 * MM;
  constexpr int NIT = RowSched<WF, 8, H1, HS / 2>::NIT;
  float w2r[MM];
#pragma unroll
  for (int t = 0; t < MM; ++t) w2r[t] = wl[2 * t + par];
  const float2* corner = halo + (q[0] * H1 + q[1]) * HS + q[2] + par;
#pragma unroll
  for (int k = 0; k < NIT; ++k) {
    const unsigned e = sch[k];
    if (e == 0xffffu) continue;
    const int t0 = e >> 8, t1 = e & 0xff;
    const float2* row = corner + (t0 * H1 + t1) * HS;
    float sre = 0, sim = 0;
#pragma unroll
    for (int t = 0; t < MM; ++t) {
      const float2 v = row[2 * t];
      sre = fmaf(w2r[t], v.x, sre);
      sim = fmaf(w2r[t], v.y, sim);
    }
    const float w01 = w0[o0 + t0] * w1[o1 + t1];
    are = fmaf(w01, sre, are);
    aim = fmaf(w01, sim, aim);
  }
}

constexpr int INTERP_NB = 32;

template <typename R, int D, int MM>
__global__ void __launch_bounds__(512)
k_interp(const __grid_constant__ CUtensorMap tmap, const cplx_t<R>* __restrict__ gp,
         cplx_t<R>* __restrict__ fout, const double* __restrict__ xs, const int* __restrict__ perm,
         const int4* __restrict__ subs, Geom g) {
  using C = cplx_t<R>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int m = MM ? MM : g.m;
  const int K = 2 * m + 1;
  const int HS = g.HS;
  const int H0 = g.H[0], H1 = D > 2 ? g.H[1] : 1;
  const int rows = D == 1 ? 1 : (D == 2 ? H0 : H0 * H1);
  const size_t hbytes = a16((size_t)rows * HS * sizeof(C));
  C* halo = reinterpret_cast<C*>(smem);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + hbytes);
  unsigned char* bufbase = smem + hbytes + 16;
  const size_t bb = batch_bytes_of(D, INTERP_NB, K, sizeof(C));
  constexpr int TEAM = InterpTeam<D, MM>::value;
  constexpr int NPW = 32 / TEAM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int tl = lane % TEAM, sub = lane / TEAM;
  const int4 sp = subs[blockIdx.x];
  int tc[D];
  tile_of<D>(g, sp.x, tc);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, (unsigned)((size_t)rows * HS * sizeof(C)));
    if constexpr (D == 1) {
      bulk_g2s(halo, gp + tc[0] * g.T[0], (unsigned)(HS * sizeof(C)), bar);
    } else {
      // padded-grid origin of the halo is tile * T; innermost coordinate in
      // 8-byte units (complex128 = two float64)
      int c[3];
      const int scale = sizeof(C) / 8;
#pragma unroll
      for (int i = 0; i < D; ++i) c[D - 1 - i] = tc[i] * g.T[i];
      c[0] *= scale;
      tma_load_box<D>(halo, &tmap, c, bar);
    }
  }
  const int end = sp.y + sp.z;
  issue_batch<C, D>(g, xs, perm, nullptr, sp.y, min(INTERP_NB, sp.z), INTERP_NB,
                    batch_at<C, D>(bufbase, INTERP_NB, K));
  cp_async_commit();
  int k = 0;
  for (int base = sp.y; base < end; base += INTERP_NB, ++k) {
    const int nb = min(INTERP_NB, end - base);
    const Batch<C, D> cur = batch_at<C, D>(bufbase + (k & 1) * bb, INTERP_NB, K);
    cp_async_wait_all();
    __syncthreads();
    finish_batch<C, D>(g, tc, nb, INTERP_NB, 1, cur);
    __syncthreads();
    if (base + INTERP_NB < end) {
      issue_batch<C, D>(g, xs, perm, nullptr, base + INTERP_NB, min(INTERP_NB, end - base - INTERP_NB),
                        INTERP_NB, batch_at<C, D>(bufbase + ((k + 1) & 1) * bb, INTERP_NB, K));
      cp_async_commit();
    }
    if (k == 0) mbar_wait(bar, 0);
    for (int j0 = warp * NPW; j0 < nb; j0 += nwarps * NPW) {
      const int jb = j0 + sub;
      const bool active = jb < nb;
      const int* q = cur.hw + (active ? jb : j0) * (2 * D + 2);
      const double* w = cur.w + (active ? jb : j0) * psi_row(D, K);
      R are = 0, aim = 0;
      if (active)
        interp_node<R, D, MM, TEAM>(halo, HS, H1, K, q, w, w + K, w + (D - 1) * K, 0, 0, tl, are, aim);
#pragma unroll
      for (int o = TEAM / 2; o; o >>= 1) {
        are += __shfl_xor_sync(0xffffffffu, are, o);
        aim += __shfl_xor_sync(0xffffffffu, aim, o);
      }
      if (tl == 0 && active) {
        C v;
        v.x = are;
        v.y = aim;
        fout[cur.pb[jb]] = v;
      }
    }
  }
}

// ---------------------------------------- B': pipelined interpolation
// PRE_PSI (tensor) mode, d = 2 / 3.  Persistent CTAs walk their
// subproblems; the halo of each comes by one TMA tensor copy (double
// buffered when two halos fit, so the next halo loads under the current
// tile), node batches (PRE_PSI rows, stencil records, output indices) by TMA
// bulk copies on an mbarrier ring refilled by thread 0 -- no coordinate
// loads, no stencil arithmetic, one CTA barrier per tile instead of two per
// batch.  Per node the TEAM-lane gather of interp_node.
struct StageMetaI {
  int nb;    // nodes (< 0: end of work)
  int last;  // last batch of its subproblem
  int poff;  // output-index offset inside the stage (alignment of the bulk copy)
  int pad;
};

template <typename R, int D, int MM>
struct IPipeCfg {
  static constexpr int K = 2 * MM + 1;
  static constexpr int H0 = D == 3 ? 8 + K : 32;
  static constexpr int H1 = D == 3 ? 8 + K : 1;
  static constexpr int HL = 8 + K;                      // last-dim halo edge
  static constexpr int ELEM = 2 * (int)sizeof(R);
  static constexpr int HS = ELEM == 8 ? HL + (HL & 1) : HL;
  static constexpr int ROWS = H0 * H1;
  // d = 3, m <= 4: two CTAs per SM.  complex64: two halos are 79 KB, so two
  // 12-warp CTAs with double-buffered halos fit (24 warps instead of 16 on
  // one 16-warp CTA).  complex128: two 8-warp CTAs with one 79 KB halo buffer
  // each -- the same 16 warps, but while one CTA sits at its tile barrier or
  // waits for its halo the other gathers, and the 32-node passes leave fewer
  // team slots empty in a subproblem's last batch than 64-node ones
  // (C5 interp: c64 12.6 -> 10.4 ms, c128 19.96 -> 18.97 ms).
#ifdef NFFTK_NO_I2CTA
  static constexpr bool TWO_CTA = false;
#else
  // complex64 at m >= 5 (one 74 KB halo buffer per CTA, 10 warps each): C3
  // c64 interp 0.207 -> 0.191 ms; complex128 at m >= 5 has 148 KB halos
  static constexpr bool TWO_CTA = D == 3 && MM > 0 && (MM <= 4 || ELEM == 8);
#endif
  // d = 2: halos and ring take 51 KB, so four 8-warp CTAs fit once the
  // registers are capped at 64 (96 / two CTAs before): C4 interp 2.23 -> 1.87
  // ms (c64 1.39 -> 1.25; a cap for three CTAs: 1.96 / 1.39)
#ifndef NFFTK_I2_BLK
#define NFFTK_I2_BLK 4
#endif
  static constexpr int BLK = TWO_CTA ? 2 : (D == 2 ? NFFTK_I2_BLK : 1);
#ifndef NFFTK_IT_C64
#define NFFTK_IT_C64 384
#endif
#ifndef NFFTK_IT_C128
#define NFFTK_IT_C128 320
#endif
#ifdef NFFTK_ITHREADS3
  static constexpr int THREADS = D == 3 ? NFFTK_ITHREADS3 : 256;
#else
  // d = 3, m >= 5 (one halo buffer): 20 warps hide more of the halo-cell
  // load latency (C3 interp 0.363 -> 0.351 ms, c64 0.230 -> 0.217; 24 warps
  // at the 85-register cap: 0.368); m <= 4 stays at 16 (C5 20.0 vs 20.5 ms)
  static constexpr int THREADS =
      D == 3 ? (MM >= 5 ? (TWO_CTA ? 320 : 640) : (TWO_CTA ? (ELEM == 8 ? NFFTK_IT_C64 : NFFTK_IT_C128) : 512)) : 256;
#endif
  // c64 d = 3: half-row lanes (interp_node3_half), teams of 16
#ifdef NFFTK_NO_HALF
  static constexpr bool HALF = false;
#else
  // HS / 2 = m + 5 must be odd; below m = 6 the half rows are too short to pay (C5 c64: 16.6 -> 21.2 ms)
  static constexpr bool HALF = D == 3 && ELEM == 8 && MM >= 6 && (MM % 2 == 0);
#endif
  static constexpr int TEAM = HALF ? 16 : InterpTeam<D, MM>::value;
  // conflict-free row schedule: d = 3, c128, 2m not a multiple of 8
#ifdef NFFTK_NO_SCHED
  static constexpr bool SCHED = false;
#else
  static constexpr bool SCHED = D == 3 && ELEM == 16 && MM > 0 && (2 * MM) % 8 != 0;
#endif
  static constexpr int NPASS = (32 / TEAM) * (THREADS / 32);  // nodes per CTA pass
  static constexpr int NB = NPASS < 16 ? 16 : (NPASS > 64 ? 64 : NPASS);
  // PRE_PSI row: halo-indexed for d = 3 ([H0 | H1 | 2m+1]), stencil-indexed
  // for d = 2 ([2m+1 | 2m+1]; halo-indexed rows would cost bytes there)
  // factor type: fp64 rows for c128, fp32 rows for c64 (k_build_psi<float>),
  // each row padded to 16 bytes
  using W = R;
  // d = 3: sten3 blocks or halo-indexed rows [H0 | H1 | 2m+1] (common.cuh
  // pipe_sten3, the layout the plan built); d = 2: stencil rows [2m+1 | 2m+1]
  static constexpr bool STEN3 = D == 3 && pipe_sten3(sizeof(R) == 4, MM);
  static constexpr bool HALO_IDX = D == 3 && !STEN3;  // leading-dim factors at their halo cell
  static constexpr int PR = psi_row_pad<W>(D == 2 ? 2 * K : (STEN3 ? sten3_count(K) : H0 + H1 + K));
  static constexpr int OW0 = STEN3 ? sten3_ow0(K) : 0, OW1 = STEN3 ? sten3_ow1(K) : (D == 3 ? H0 : 0),
                       OWL = STEN3 ? STEN3_OW2 : (D == 3 ? H0 + H1 : K);
  static constexpr size_t al(size_t v) { return (v + 15) & ~(size_t)15; }
  static constexpr size_t W_BYTES = al(sizeof(W) * NB * PR);
  static constexpr size_t R_BYTES = al(16 * (size_t)NB);
  static constexpr size_t SB = W_BYTES + R_BYTES + al(4 * (size_t)(NB + 4));
  static constexpr size_t al128(size_t v) { return (v + 127) & ~(size_t)127; }
  static constexpr size_t HALO = al128((size_t)ROWS * HS * ELEM);  // TMA tensor destinations: 128 B
  static constexpr size_t ctl_bytes(int s) { return al(16 * (size_t)s + sizeof(StageMetaI) * s + 64 + 16); }
  static constexpr size_t halo_off(int s) { return al128(s * SB + ctl_bytes(s)); }
  static constexpr size_t LIMIT = TWO_CTA ? 112 * 1024 : 224 * 1024;
  // prefer double-buffered halos (next halo loads under the current tile),
  // then the deepest node ring
  static constexpr int pick_s() {
    for (int s : {4, 3, 2})
      if (halo_off(s) + 2 * HALO <= LIMIT) return s;
    for (int s : {4, 3})
      if (halo_off(s) + HALO <= LIMIT) return s;
    return 2;
  }
  static constexpr int S = pick_s();
  static constexpr size_t CTL = S * SB;
  static constexpr size_t CTL_BYTES = ctl_bytes(S);
  static constexpr size_t HALO_OFF = halo_off(S);
  static constexpr int NH = HALO_OFF + 2 * HALO <= LIMIT ? 2 : 1;
  static constexpr size_t SMEM = HALO_OFF + NH * HALO;
};

template <typename R, int D, int MM>
__global__ void __launch_bounds__(IPipeCfg<R, D, MM>::THREADS, IPipeCfg<R, D, MM>::BLK)
k_interp_pipe(const __grid_constant__ CUtensorMap tmap, cplx_t<R>* __restrict__ fout,
              const double* __restrict__ psi, const int4* __restrict__ rec,
              const int* __restrict__ perm, const int4* __restrict__ subs, int nsubs, Geom g) {
  using C = cplx_t<R>;
  using P = IPipeCfg<R, D, MM>;
  constexpr int K = P::K, HS = P::HS, H1 = P::H1, PR = P::PR, NB = P::NB, S = P::S, NH = P::NH;
  constexpr int TEAM = P::TEAM, NPW = 32 / TEAM, NW = P::THREADS / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + P::CTL);
  unsigned long long* empty = full + S;
  unsigned long long* hbar = empty + S;  // NH halo barriers
  StageMetaI* meta = reinterpret_cast<StageMetaI*>(hbar + 2);
  int* pst = reinterpret_cast<int*>(meta + S);  // producer: s, base, end, k, drawn, seq
  int* subq = pst + 6;                           // the CTA's subproblem sequence (ring of 8)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tl = lane % TEAM, sub = lane / TEAM;
  const unsigned halo_tx = (unsigned)(P::ROWS * HS * sizeof(C));
  constexpr int NIT = P::SCHED  ? RowSched<2 * (MM > 0 ? MM : 1), TEAM, H1, HS>::NIT
                     : P::HALF ? RowSched<2 * (MM > 0 ? MM : 1), 8, H1, HS / 2>::NIT
                               : 1;
  unsigned sch[NIT];
  if constexpr (P::SCHED) {
#pragma unroll
    for (int k = 0; k < NIT; ++k)
      sch[k] = c_row_sched<2 * (MM > 0 ? MM : 1), TEAM, H1, HS>.v[k * TEAM + tl];
  } else if constexpr (P::HALF) {
#pragma unroll
    for (int k = 0; k < NIT; ++k)
      sch[k] = c_row_sched<2 * (MM > 0 ? MM : 1), 8, H1, HS / 2>.v[k * 8 + (tl >> 1)];
  }
  auto issue_halo = [&](int s, int buf) {
    int tc[D];
    tile_of<D>(g, subs[s].x, tc);
    int c[3];
    const int scale = sizeof(C) / 8;
#pragma unroll
    for (int i = 0; i < D; ++i) c[D - 1 - i] = tc[i] * g.T[i];
    c[0] *= scale;
    mbar_expect_tx(hbar + buf, halo_tx);
    tma_load_box<D>(smem + P::HALO_OFF + buf * P::HALO, &tmap, c, hbar + buf);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, NW);
    }
    for (int i = 0; i < NH; ++i) mbar_init(hbar + i, 1);
    pst[0] = blockIdx.x;
    pst[3] = 0;
    pst[4] = 1;  // subproblems drawn (the first is blockIdx.x)
    pst[5] = 0;  // producer's position in the sequence
    subq[0] = blockIdx.x;
    if (blockIdx.x < nsubs) {
      const int4 sp = subs[blockIdx.x];
      pst[1] = sp.y;
      pst[2] = sp.y + sp.z;
    }
  }
  __syncthreads();
  // j-th subproblem of this CTA (thread 0 only): producer and halo issue walk
  // the same sequence; dynamic tickets (next_sub), no draw past the end
  auto sub_at = [&](int j) {
    while (pst[4] <= j) {
      const int prev = subq[(pst[4] - 1) & 7];
      subq[pst[4] & 7] = prev >= nsubs ? prev : next_sub(g, SCHED_INTERP, prev);
      ++pst[4];
    }
    return subq[j & 7];
  };
  auto produce = [&]() {
    const int pk = pst[3];
    const int slot = pk % S;
    if (pk >= S) mbar_wait(empty + slot, ((pk / S) - 1) & 1);
    StageMetaI* mt = meta + slot;
    pst[3] = pk + 1;
    if (pst[0] >= nsubs) {
      mt->nb = -1;
      mbar_arrive(full + slot);
      return;
    }
    const int pbase = pst[1], pend = pst[2];
    const int nb = min(NB, pend - pbase);
    const int poff = pbase & 3;
    const int pcnt = (nb + poff + 3) & ~3;
    mt->nb = nb;
    mt->last = pbase + nb >= pend;
    mt->poff = poff;
    unsigned char* st = smem + slot * P::SB;
    const unsigned wb = (unsigned)(sizeof(typename P::W) * PR) * nb, rb = 16u * nb, pb = 4u * pcnt;
    mbar_expect_tx(full + slot, wb + rb + pb);
#ifdef NFFTK_NO_STREAM_HINT
    bulk_g2s(st, reinterpret_cast<const typename P::W*>(psi) + (int64_t)pbase * PR, wb, full + slot);
    bulk_g2s(st + P::W_BYTES, rec + pbase, rb, full + slot);
    bulk_g2s(st + P::W_BYTES + P::R_BYTES, perm + (pbase - poff), pb, full + slot);
#else
    // streamed once: L2 evict-first keeps the halo boxes the tiles share resident
    const unsigned long long pol = l2_evict_first_policy();
    bulk_g2s_stream(st, reinterpret_cast<const typename P::W*>(psi) + (int64_t)pbase * PR, wb, full + slot, pol);
    bulk_g2s_stream(st + P::W_BYTES, rec + pbase, rb, full + slot, pol);
    bulk_g2s_stream(st + P::W_BYTES + P::R_BYTES, perm + (pbase - poff), pb, full + slot, pol);
#endif
    if (pbase + nb < pend) {
      pst[1] = pbase + nb;
    } else {
      const int s = sub_at(++pst[5]);
      pst[0] = s;
      if (s < nsubs) {
        const int4 sp = subs[s];
        pst[1] = sp.y;
        pst[2] = sp.y + sp.z;
      }
    }
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < S - 1; ++i) produce();
    if (NH == 2 && (int)blockIdx.x < nsubs) issue_halo(blockIdx.x, 0);
  }
  int k = 0;
  for (int it = 0;; ++it) {  // subproblems of this CTA, in sub_at order
    const int buf = NH == 2 ? (it & 1) : 0;
    __syncthreads();  // every warp is done with the halo buffer about to be refilled
    if (threadIdx.x == 0) {
      if constexpr (NH == 1) {
        const int s = sub_at(it);
        if (s < nsubs) issue_halo(s, 0);
#ifndef NFFTK_NO_HALO_L2PF
        // the next halo is pulled into L2 under this tile (one buffer: its
        // shared-memory load has to wait for the tile to end; C3 interp
        // 0.343 -> 0.339 ms)
        if constexpr (D == 3) {
          const int s2 = sub_at(it + 1);
          if (s2 < nsubs) {
            int tc[3], c[3];
            tile_of<3>(g, subs[s2].x, tc);
            for (int i = 0; i < 3; ++i) c[2 - i] = tc[i] * g.T[i];
            c[0] *= (int)(sizeof(C) / 8);
            tma_prefetch_box3(&tmap, c);
          }
        }
#endif
      } else {
        const int s = sub_at(it + 1);
        if (s < nsubs) issue_halo(s, buf ^ 1);
      }
    }
    // the ring says whether a subproblem follows (end marker: no halo was issued)
    mbar_wait(full + k % S, (k / S) & 1);
    if (meta[k % S].nb < 0) break;
    mbar_wait(hbar + buf, (NH == 2 ? (it >> 1) : it) & 1);
    const C* halo = reinterpret_cast<const C*>(smem + P::HALO_OFF + buf * P::HALO);
    for (;; ++k) {  // batches of the subproblem
      const int slot = k % S;
      mbar_wait(full + slot, (k / S) & 1);
      const StageMetaI mt = meta[slot];
      const unsigned char* st = smem + slot * P::SB;
      const typename P::W* ws = reinterpret_cast<const typename P::W*>(st);
      const int4* rs = reinterpret_cast<const int4*>(st + P::W_BYTES);
      const int* pv = reinterpret_cast<const int*>(st + P::W_BYTES + P::R_BYTES) + mt.poff;
      for (int j0 = warp * NPW; j0 < mt.nb; j0 += NW * NPW) {
        const int jb = j0 + sub;
        const bool active = jb < mt.nb;
        const int jj = active ? jb : j0;
        const int4 r = rs[jj];
        const unsigned wp = (unsigned)r.w;
        int q[8];
        q[0] = r.x;
        q[1] = r.y;
        if constexpr (D == 3) {
          q[2] = r.z;
          q[3] = wp & 0xff;
          q[4] = (wp >> 8) & 0xff;
          q[5] = (wp >> 16) & 0xff;
          q[6] = (wp >> 24) & 1;
        } else {
          q[2] = wp & 0xff;
          q[3] = (wp >> 8) & 0xff;
          q[4] = (wp >> 24) & 1;
        }
        R are = 0, aim = 0;
        // complex64 8-lane teams (interp_node): the odd team of a half warp
        // walks its rows rotated when the pair's last-dim starts share parity
        int sh = 0;
        if constexpr (D == 3 && sizeof(R) == 4 && TEAM == 8 && !P::HALF) {
          const int q2p = __shfl_xor_sync(0xffffffffu, q[2], 8);
          sh = ((lane >> 3) & 1) & ~((q[2] ^ q2p) & 1) & (int)q[6];
#ifdef NFFTK_NO_ROT
          sh = 0;
#endif
        }
        if (active) {
          const typename P::W* w = ws + jj * PR;
          // factor blocks: leading dims at w + OW0 / OW1 (indexed from the
          // node's stencil start o0 / o1 for halo-indexed rows, from 0
          // otherwise), last dim at w + OWL
          const int o0 = P::HALO_IDX ? q[0] : 0, o1 = P::HALO_IDX ? q[1] : 0;
          if constexpr (D == 3 && P::SCHED) {
            if (q[6])  // fast node: conflict-free row schedule
              interp_node3_sched<MM, TEAM, H1, HS>(reinterpret_cast<const double2*>(halo), q, w + P::OW0,
                                                   w + P::OW1, w + P::OWL, o0, o1, sch, are, aim);
            else
              interp_node<R, D, MM, TEAM>(halo, HS, H1, K, q, w + P::OW0, w + P::OW1, w + P::OWL, o0, o1,
                                          tl, are, aim);
          } else if constexpr (D == 3 && P::HALF) {
            if (q[6])  // fast node: half-row lanes on the conflict-free schedule
              interp_node3_half<MM, H1, HS>(reinterpret_cast<const float2*>(halo), q, w + P::OW0,
                                            w + P::OW1, w + P::OWL, o0, o1, tl & 1, sch, are, aim);
            else
              interp_node<R, D, MM, TEAM>(halo, HS, H1, K, q, w + P::OW0, w + P::OW1, w + P::OWL, o0, o1,
                                          tl, are, aim);
          } else if constexpr (D == 3)
            interp_node<R, D, MM, TEAM>(halo, HS, H1, K, q, w + P::OW0, w + P::OW1, w + P::OWL, o0, o1,
                                        tl, are, aim, sh);
          else  // stencil-indexed rows [2m+1 | 2m+1]
            interp_node<R, D, MM, TEAM>(halo, HS, H1, K, q, w, w, w + K, 0, 0, tl, are, aim);
        }
#pragma unroll
        for (int o = TEAM / 2; o; o >>= 1) {
          are += __shfl_xor_sync(0xffffffffu, are, o);
          aim += __shfl_xor_sync(0xffffffffu, aim, o);
        }
        if (tl == 0 && active) {
          C v;
          v.x = are;
          v.y = aim;
          fout[pv[jb]] = v;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
      if (threadIdx.x == 0) produce();
      if (mt.last) {
        ++k;
        break;
      }
    }
  }
  if (threadIdx.x == 0) sched_done(g, SCHED_INTERP);
}

// Dynamic tickets pay where a CTA walks many subproblems of uneven weight
// (clustered C4: spread 2.90 -> 2.35 ms, interp 2.59 -> 2.41); with a
// handful per CTA (C2: 1.5 per spread CTA, 12 per interp CTA) the ticket
// latency on the producer's and halo issue's path costs more than the
// balance gains (C2 step 0.120 -> 0.126 ms with dynamic interp tickets).
static Geom sched_geom(const Geom& g, int nsubs, int grid, int per_cta = 4) {
  Geom q = g;
  if ((int64_t)nsubs < (int64_t)per_cta * grid) q.sched = nullptr;
  return q;
}

// Geometries the pipelined kernels (spread and interp) both cover; for d = 3
// these get the pipelined PRE_PSI layouts (Geom::psi_pad, common.cuh pipe_sten3).
bool pipe_geometry(const Geom& g) {
  if (getenv("NFFTK_NO_PIPE")) return false;
  if (g.d == 3) return g.m >= 1 && g.m <= 6 && g.T[0] == 8 && g.T[1] == 8 && g.T[2] == 8;
  if (g.d == 2) return g.m >= 1 && g.m <= 8 && g.H[0] == 32 && g.T[1] == 8;
  return false;
}

bool interp_pipe_ok(const Geom& g) {
  return g.mode == MODE_TENSOR && g.psi && g.rec && pipe_geometry(g) && (g.psi_pad != 0) == (g.d == 3);
}

// Sorted copy of the samples for the spread: fs[i] = f[perm[i]].
template <typename C>
__global__ void k_permute_samples(const C* __restrict__ f, const int* __restrict__ perm, int64_t M,
                                  C* __restrict__ fs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x)
    fs[i] = f[perm[i]];
}

// =========================================================== B^H: spreading
// Shared-memory halo accumulation without atomics: halo cells are owned by
// warps through their absolute halo row index (d=3: a mod UA with UA = 2m,
// so a generic node gives every warp exactly one a-row; d=2: half-warps own
// a mod U; d=1: threads own cells mod U), so two warps never touch the same
// cell -- the GPU form of the reference's slab ownership (kernels.py:13-17).
// Per batch the CTA stages, for every node, the complex row coefficients
// f_j * w0[t] and (d=3, generic nodes) the w1 (x) w2 factor plane, so each
// warp's per-node work is a handful of loads plus one 5-instruction
// read-modify-write per cell.  The finished halo is added to the padded HBM
// grid with TMA bulk reductions, one per halo row.
template <typename R, int D, int MM>
__global__ void __launch_bounds__(512)
k_spread(cplx_t<R>* __restrict__ gp, const cplx_t<R>* __restrict__ fsorted,
         const double* __restrict__ xs, const int4* __restrict__ subs, Geom g) {
  using C = cplx_t<R>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int m = MM ? MM : g.m;
  const int K = 2 * m + 1;
  constexpr int WF = 2 * (MM > 0 ? MM : 1);
  const int NB = g.nb_spread;
  const int HS = g.HS;
  const int H0 = g.H[0], H1 = D > 2 ? g.H[1] : 1;
  const int rows = D == 1 ? 1 : (D == 2 ? H0 : H0 * H1);
  const int hsz = rows * HS;
  size_t off = 0;
  C* halo = reinterpret_cast<C*>(smem);
  off += a16((size_t)hsz * sizeof(C));
  C* coef = reinterpret_cast<C*>(smem + off);          // [NB][K]  f * w0[t]
  off += a16((size_t)NB * K * sizeof(C));
  double* plane = reinterpret_cast<double*>(smem + off);  // [NB][WF*WF] (d=3)
  off += D == 3 ? a16((size_t)NB * WF * WF * sizeof(double)) : 0;
  unsigned char* bufbase = smem + off;
  const size_t bb = batch_bytes_of(D, NB, K, sizeof(C));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int4 sp = subs[blockIdx.x];
  int tc[D];
  tile_of<D>(g, sp.x, tc);
  const int end = sp.y + sp.z;
  issue_batch<C, D>(g, xs, nullptr, fsorted, sp.y, min(NB, sp.z), NB, batch_at<C, D>(bufbase, NB, K));
  cp_async_commit();
  for (int idx = threadIdx.x; idx < hsz; idx += blockDim.x) {
    C z;
    z.x = 0;
    z.y = 0;
    halo[idx] = z;
  }
  const int UA = D == 3 ? nwarps : 1;
  // per-lane cell offsets inside a node's (b, c) plane, fast path (d=3)
  constexpr int NK = (WF * WF + 31) / 32;
  int offk[NK];
#pragma unroll
  for (int kk = 0; kk < NK; ++kk) {
    int p = lane + 32 * kk;
    int t1 = p / WF, t2 = p - t1 * WF;
    offk[kk] = t1 * HS + t2;
  }
  int k = 0;
  for (int base = sp.y; base < end; base += NB, ++k) {
    const int nb = min(NB, end - base);
    const Batch<C, D> cur = batch_at<C, D>(bufbase + (k & 1) * bb, NB, K);
    cp_async_wait_all();
    __syncthreads();  // batch k landed; previous batch applied; zeroing done
    finish_batch<C, D>(g, tc, nb, NB, UA, cur);
    __syncthreads();
    // derived per-node data: row coefficients, factor plane
    for (int q = threadIdx.x; q < nb * K; q += blockDim.x) {
      int j = q / K, t = q - j * K;
      R w0 = (R)cur.w[j * psi_row(D, K) + t];
      C f = cur.fv[j];
      C c;
      c.x = f.x * w0;
      c.y = f.y * w0;
      coef[q] = c;
    }
    if constexpr (D == 3) {
      if (MM > 0) {
        for (int q = threadIdx.x; q < nb * WF * WF; q += blockDim.x) {
          int j = q / (WF * WF), p = q - j * (WF * WF), t1 = p / WF, t2 = p - t1 * WF;
          plane[q] = cur.w[j * psi_row(D, K) + K + t1] * cur.w[j * psi_row(D, K) + 2 * K + t2];
        }
      }
    }
    __syncthreads();
    if (base + NB < end) {
      issue_batch<C, D>(g, xs, nullptr, fsorted, base + NB, min(NB, end - base - NB), NB,
                        batch_at<C, D>(bufbase + ((k + 1) & 1) * bb, NB, K));
      cp_async_commit();
    }
    if constexpr (D == 3) {
      for (int jb = 0; jb < nb; ++jb) {
        const int* q = cur.hw + jb * (2 * D + 2);
        const int h0 = q[0];
        int d0 = warp - q[7];
        if (d0 < 0) d0 += UA;
        if (MM > 0 && q[6] && UA == WF) {
          // generic node: exactly one owned row a = h0 + d0
          const C cf = coef[jb * K + d0];
          C* cellp = halo + ((h0 + d0) * H1 + q[1]) * HS + q[2];
          const double* pl = plane + jb * WF * WF;
#pragma unroll
          for (int kk = 0; kk < NK; ++kk) {
            if (kk < NK - 1 || lane + 32 * kk < WF * WF) {
              R ww = (R)pl[lane + 32 * kk];
              C* cell = cellp + offk[kk];
              C v = *cell;
              v.x = fma(cf.x, ww, v.x);
              v.y = fma(cf.y, ww, v.y);
              *cell = v;
            }
          }
        } else {
          const int h1 = q[1], h2 = q[2], W0 = q[3], W1 = q[4], W2 = q[5];
          const double* w = cur.w + jb * psi_row(D, K);
          for (int a = h0 + d0; a < h0 + W0; a += UA) {
            const C cf = coef[jb * K + (a - h0)];
            C* pl = halo + (a * H1 + h1) * HS + h2;
            for (int p = lane; p < W1 * W2; p += 32) {
              int t1 = p / W2, t2 = p - t1 * W2;
              R ww = (R)(w[K + t1] * w[2 * K + t2]);
              C* cell = pl + t1 * HS + t2;
              C v = *cell;
              v.x = fma(cf.x, ww, v.x);
              v.y = fma(cf.y, ww, v.y);
              *cell = v;
            }
          }
        }
        __syncwarp();
      }
    } else {
      // d = 1, 2: the CTA is one warp with a private halo; one node at a time,
      // lanes over the node's stencil cells (distinct cells, no conflicts)
      for (int jb = 0; jb < nb; ++jb) {
        const int* q = cur.hw + jb * (2 * D + 2);
        const double* w = cur.w + jb * psi_row(D, K);
        if constexpr (D == 2) {
          const int W0 = q[2], W1 = q[3];
          C* corner = halo + q[0] * HS + q[1];
          for (int p = lane; p < W0 * W1; p += 32) {
            int t0 = p / W1, t1 = p - t0 * W1;
            const C cf = coef[jb * K + t0];
            R ww = (R)w[K + t1];
            C* cell = corner + t0 * HS + t1;
            C v = *cell;
            v.x = fma(cf.x, ww, v.x);
            v.y = fma(cf.y, ww, v.y);
            *cell = v;
          }
        } else {
          const int W0 = q[1];
          for (int t0 = lane; t0 < W0; t0 += 32) {
            const C cf = coef[jb * K + t0];
            C* cell = halo + q[0] + t0;
            C v = *cell;
            v.x += cf.x;
            v.y += cf.y;
            *cell = v;
          }
        }
        __syncwarp();
      }
    }
  }
  // ---- flush: one TMA bulk reduction per halo row into the padded grid
  fence_proxy_async_smem();
  __syncthreads();
  for (int r = threadIdx.x; r < rows; r += blockDim.x) {
    int64_t row0;
    if constexpr (D == 1) {
      row0 = (int64_t)tc[0] * g.T[0];
    } else if constexpr (D == 2) {
      row0 = (int64_t)(tc[0] * g.T[0] + r) * g.np[1] + tc[1] * g.T[1];
    } else {
      int a = r / H1, b = r - a * H1;
      row0 = ((int64_t)(tc[0] * g.T[0] + a) * g.np[1] + tc[1] * g.T[1] + b) * g.np[2] + tc[2] * g.T[2];
    }
    bulk_red_add<R>(gp + row0, halo + (size_t)r * HS, (unsigned)(HS * sizeof(C)));
  }
  bulk_commit_wait_read();
}

// ============================================ B^H, d = 3: register-resident
// Each thread owns one full halo row (a, b): all H2 = T2 + 2m + 1 cells of it
// live in registers.  A node's c-offset h2 (and its stencil rows) are the
// same for every thread, so the c-run of a node is added with a switch on
// h2 whose bodies index the register row statically -- no shared-memory
// read-modify-write, no ownership bookkeeping, no conflicts (each cell has
// exactly one owner).  A warp skips nodes whose stencil misses all its rows.
// Zero-padded K = 2m+1 factor rows make grid-aligned nodes (width 2m+1) take
// the same path.  At the end the rows go through shared memory and are
// added to the padded grid by TMA bulk reductions.
template <int MM, int T2>
struct RRThreads {
  static constexpr int value = (((T2 + 2 * MM + 1) * (T2 + 2 * MM + 1)) + 31) / 32 * 32;
  // CTAs per SM the register budget allows (accumulator rows dominate)
  static constexpr int blocks = value * 2 * 102 <= 65536 && MM <= 4 ? 2 : 1;
};

template <typename R, int MM, int T2>
__global__ void __launch_bounds__(RRThreads<MM, T2>::value, RRThreads<MM, T2>::blocks)
k_spread_rr(cplx_t<R>* __restrict__ gp, const cplx_t<R>* __restrict__ fsorted,
            const double* __restrict__ xs, const int4* __restrict__ subs, int nsubs, Geom g) {
  using C = cplx_t<R>;
  constexpr int K = 2 * MM + 1;
  constexpr int H2 = T2 + 2 * MM + 1;
  extern __shared__ __align__(128) unsigned char smem[];
  const int NB = g.nb_spread;
  const int H1 = g.H[1];
  const int HS = g.HS;
  const int rows = g.H[0] * H1;
  size_t off = 0;
  C* stage = reinterpret_cast<C*>(smem);  // per-thread staging rows for the bulk reductions
  off += a16((size_t)rows * HS * sizeof(C));
  C* coef = reinterpret_cast<C*>(smem + off);  // [NB][K]  f * w0[t]
  off += a16((size_t)NB * K * sizeof(C));
  unsigned char* bufbase = smem + off;
  const size_t bb = batch_bytes_of(3, NB, K, sizeof(C));
  int s = blockIdx.x;
  if (s >= nsubs) return;
  int4 sp = subs[s];
  int tc[3];
  tile_of<3>(g, sp.x, tc);
  issue_batch<C, 3>(g, xs, nullptr, fsorted, sp.y, min(NB, sp.z), NB, batch_at<C, 3>(bufbase, NB, K));
  cp_async_commit();
  // strided row ownership: warp w, lane l owns halo row l * nw + w, so every
  // warp holds a mix of centre rows (hit by most nodes) and edge rows (hit by
  // few) -- equal work per warp, no batch-barrier imbalance
  const int nw = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int row = lane * nw + (threadIdx.x >> 5);
  const bool owner = row < rows;
  const int a = owner ? row / H1 : 0, b = owner ? row - (row / H1) * H1 : 0;
  R accr[H2], acci[H2];
#pragma unroll
  for (int c = 0; c < H2; ++c) accr[c] = acci[c] = 0;
  bool touched = false;
  int base = sp.y;
  for (int k = 0;; ++k) {
    const int end = sp.y + sp.z;
    const int nb = min(NB, end - base);
    const Batch<C, 3> cur = batch_at<C, 3>(bufbase + (k & 1) * bb, NB, K);
    // next (subproblem, batch) item of this persistent CTA
    int s_n = s, base_n = base + NB;
    int4 sp_n = sp;
    if (base_n >= end) {
      s_n = s + gridDim.x;
      if (s_n < nsubs) {
        sp_n = subs[s_n];
        base_n = sp_n.y;
      }
    }
    cp_async_wait_all();
    __syncthreads();
    finish_batch<C, 3>(g, tc, nb, NB, 1, cur);
    if (g.mode != MODE_TENSOR) __syncthreads();  // computed factors feed the coefficients
    for (int q = threadIdx.x; q < nb * K; q += blockDim.x) {
      int j = q / K, t = q - j * K;
      R w0 = (R)cur.w[j * psi_row(3, K) + t];
      C f = cur.fv[j];
      C c;
      c.x = f.x * w0;
      c.y = f.y * w0;
      coef[q] = c;
    }
    __syncthreads();
    if (s_n < nsubs) {
      issue_batch<C, 3>(g, xs, nullptr, fsorted, base_n, min(NB, sp_n.y + sp_n.z - base_n), NB,
                        batch_at<C, 3>(bufbase + ((k + 1) & 1) * bb, NB, K));
      cp_async_commit();
    }
    if (!(g.debug & 2)) {
      for (int jb = 0; jb < nb; ++jb) {
        const int* q = cur.hw + jb * 8;
        const int4 qa = *reinterpret_cast<const int4*>(q);  // h0, h1, h2, W0
        const int W1 = q[4];
        const int ta = a - qa.x, tb = b - qa.y;
        const bool act = owner && ta >= 0 && ta < qa.w && tb >= 0 && tb < W1;
        const double* w = cur.w + jb * psi_row(3, K);
        R cr = 0, ci = 0;
        if (act) {
          const C cf = coef[jb * K + ta];
          R w1 = (R)w[K + tb];
          cr = cf.x * w1;
          ci = cf.y * w1;
          touched = true;
        }
        // c-run factors: preloaded into a register array for small m (latency
        // off the FMA chain), loaded inside the case for large m (register
        // pressure at 1 CTA/SM); measured both ways on C3 (m=6) and C5 (m=4)
#define NFFTK_RR_CASE(H, WT)                                       \
  case H:                                                          \
    if constexpr (H + K <= H2) {                                   \
      _Pragma("unroll") for (int t = 0; t < K; ++t) {              \
        accr[H + t] = fma(cr, WT, accr[H + t]);                    \
        acci[H + t] = fma(ci, WT, acci[H + t]);                    \
      }                                                            \
    }                                                              \
    break;
#define NFFTK_RR_SWITCH(WT)                                                                      \
  switch (qa.z) {                                                                                \
    NFFTK_RR_CASE(0, WT) NFFTK_RR_CASE(1, WT) NFFTK_RR_CASE(2, WT) NFFTK_RR_CASE(3, WT)          \
    NFFTK_RR_CASE(4, WT) NFFTK_RR_CASE(5, WT) NFFTK_RR_CASE(6, WT) NFFTK_RR_CASE(7, WT)          \
    NFFTK_RR_CASE(8, WT)                                                                         \
    default: break;                                                                              \
  }
        if constexpr (MM <= 4) {
          R w2[K];
#pragma unroll
          for (int t = 0; t < K; ++t) w2[t] = (R)w[2 * K + t];
          NFFTK_RR_SWITCH(w2[t])
        } else {
          const double* w2 = w + 2 * K;
          NFFTK_RR_SWITCH((R)w2[t])
        }
#undef NFFTK_RR_SWITCH
#undef NFFTK_RR_CASE
      }
    }
    if (s_n != s) {
      // tile done: each thread stages and bulk-reduces its own row -- no CTA
      // barrier; the row slot is reused only after this thread's previous
      // reduction finished reading it
      if (owner && touched && !(g.debug & 1)) {
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        C* dst = stage + (size_t)row * HS;
#pragma unroll
        for (int c = 0; c < H2; ++c) {
          C v;
          v.x = accr[c];
          v.y = acci[c];
          dst[c] = v;
        }
        if (HS > H2) {
          C z;
          z.x = 0;
          z.y = 0;
          dst[H2] = z;
        }
        fence_proxy_async_smem();
        int64_t row0 =
            ((int64_t)(tc[0] * g.T[0] + a) * g.np[1] + tc[1] * g.T[1] + b) * g.np[2] + tc[2] * g.T[2];
        bulk_red_add<R>(gp + row0, dst, (unsigned)(HS * sizeof(C)));
        asm volatile("cp.async.bulk.commit_group;\n" ::);
      }
#pragma unroll
      for (int c = 0; c < H2; ++c) accr[c] = acci[c] = 0;
      touched = false;
      if (s_n >= nsubs) break;
      s = s_n;
      sp = sp_n;
      tile_of<3>(g, sp.x, tc);
    }
    base = base_n;
  }
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

// ------------------------------------------- C': pipelined register spread
// PRE_PSI (tensor) mode, d = 3.  Same row ownership and register
// accumulators as k_spread_rr, fed by a ring of S node-batch stages instead of
// lock-step batches:
//  * a stage is three TMA bulk copies (PRE_PSI rows, stencil records, sorted
//    samples) completing on the stage's `full` mbarrier -- no per-node
//    coordinate loads, no stencil arithmetic, no CTA barrier;
//  * each warp releases a stage on its `empty` mbarrier when done; thread 0
//    refills the stage consumed one step earlier (lag 1), so warps drift
//    freely within the ring;
//  * nodes of a tile are sorted by their last-dim stencil start (k_bin_keys),
//    so the offset switch runs once per run of equal starts, not per node.
struct StageMeta {
  int tile;  // tile of this batch
  int nb;    // nodes (< 0: end of work)
  int last;  // last batch of its tile: flush after it
  int foff;  // sample offset inside the stage (alignment of the bulk copy)
};

__host__ __device__ inline size_t pipe_stage_bytes(int nb, int K, int elem) {
  auto al = [](size_t v) { return (v + 15) & ~(size_t)15; };
  return al(sizeof(double) * nb * psi_row(3, K)) + al(16 * (size_t)nb) + al((size_t)elem * (nb + 2));
}

// Compile-time geometry of k_spread_pipe (T = 8 in every dim): halo rows,
// threads, CTAs per SM, and the largest ring (batch NB x S stages) that fits.
template <typename R, int MM>
struct PipeCfg {
  static constexpr int K = 2 * MM + 1;
  static constexpr int H = 8 + K;                        // halo edge
  static constexpr int ELEM = 2 * (int)sizeof(R);        // complex element bytes
  static constexpr int HS = ELEM == 8 ? H + 1 : H;       // row stride (Geom::HS)
  static constexpr int ROWS = H * H;
#ifndef NFFTK_RPT
#define NFFTK_RPT 1
#endif
  static constexpr int RPT = sizeof(R) == 8 ? NFFTK_RPT : 1;  // rows per thread (run-window path)
  static constexpr int HB = (H + RPT - 1) / RPT;              // row groups per a-line
  static constexpr int GROUPS = H * HB;
  static constexpr int THREADS = (GROUPS + 31) / 32 * 32;
  // two CTAs per SM: complex128 at m <= 4 (run-window accumulators, below);
  // complex64 at every m -- its whole-row accumulators are fp32 (72 registers
  // at m = 6, 80 at m = 5: no spills under the two-CTA cap) and its staging
  // rows half the size: C3 c64 spread 0.254 -> 0.188 ms
#ifdef NFFTK_NO_SPREAD_C64_2CTA
  static constexpr int BLOCKS = THREADS * 2 * 102 <= 65536 && MM <= 4 ? 2 : 1;
#else
  static constexpr int BLOCKS = (THREADS * 2 * 102 <= 65536 && MM <= 4) || sizeof(R) == 4 ? 2 : 1;
#endif
  // Register budget of 2 CTAs/SM: run-window accumulators (K cells, the
  // factor loads of a node all in flight) instead of the whole halo row
  // (measured C5 spread 52.2 -> 41.8 ms; the whole-row switch stays 5% faster
  // at m = 6 (1 CTA/SM, 128 registers) and 3% faster for fp32 rows).
  static constexpr bool RUNACC = (BLOCKS == 2 || RPT > 1) && sizeof(R) == 8;
  using W = R;                                          // factor type (fp32 rows for c64)
  // PRE_PSI row: sten3 blocks [2m+2 | 2m+2 | 2m+2] or halo-indexed [H | H | 2m+1] (pipe_sten3)
  static constexpr bool STEN3 = pipe_sten3(sizeof(R) == 4, MM);
  static constexpr int PR = psi_row_pad<W>(STEN3 ? sten3_count(K) : 2 * H + K);
  static constexpr size_t al(size_t v) { return (v + 15) & ~(size_t)15; }
  static constexpr size_t stage_bytes(int nb) {
    return al(sizeof(W) * nb * PR) + al(16 * (size_t)nb) + al((size_t)ELEM * (nb + 2));
  }
  // staging rows: one per halo row (RUNACC: RPT per row group, GROUPS * RPT may exceed ROWS)
  static constexpr size_t rows_bytes = al((size_t)(GROUPS * RPT > ROWS ? GROUPS * RPT : ROWS) * HS * ELEM);
  static constexpr size_t ctl_bytes(int s) { return al(16 * (size_t)s + sizeof(StageMeta) * s + 32); }
  static constexpr size_t total(int nb, int s) { return s * stage_bytes(nb) + ctl_bytes(s) + rows_bytes; }
  static constexpr size_t budget = BLOCKS == 2 ? 112 * 1024 : 224 * 1024;
#ifndef NFFTK_SPREAD_MINS
#define NFFTK_SPREAD_MINS 2
#endif
  // the largest batch whose ring is at least MINS deep, then the deepest ring
  static constexpr int pick_nb() {
    for (int nb : {32, 16, 8})
      for (int s : {8, 6, 5, 4, 3, 2})
        if (s >= NFFTK_SPREAD_MINS && total(nb, s) <= budget) return nb;
    return 0;
  }
  static constexpr int pick_s() {
    for (int nb : {32, 16, 8})
      for (int s : {8, 6, 5, 4, 3, 2})
        if (s >= NFFTK_SPREAD_MINS && total(nb, s) <= budget) return s;
    return 0;
  }
  static constexpr int NB = pick_nb();
  static constexpr int S = pick_s();
  static constexpr size_t SB = stage_bytes(NB > 0 ? NB : 1);
  static constexpr size_t W_BYTES = al(sizeof(W) * (NB > 0 ? NB : 1) * PR);
  static constexpr size_t R_BYTES = al(16 * (size_t)(NB > 0 ? NB : 1));
  static constexpr size_t CTL = (S > 0 ? S : 1) * SB;    // control block offset
  static constexpr size_t ROWS_OFF = CTL + ctl_bytes(S > 0 ? S : 1);
  static constexpr size_t SMEM = ROWS_OFF + rows_bytes;
};

// GATHER: warp 0 fetches the batch's samples through perm itself (lane l <
// NB: one cp.async of f[perm[base + l]] arriving on the batch's mbarrier, the
// index loaded one batch ahead) instead of reading a sorted copy (residue.cu).
template <typename R, int MM, bool GATHER>
__global__ void __launch_bounds__(PipeCfg<R, MM>::THREADS, PipeCfg<R, MM>::BLOCKS)
k_spread_pipe(cplx_t<R>* __restrict__ gp, const cplx_t<R>* __restrict__ fsorted,
              const cplx_t<R>* __restrict__ funs, const int* __restrict__ perm,
              const double* __restrict__ psi, const int4* __restrict__ rec,
              const int4* __restrict__ subs, int nsubs, Geom g) {
  using C = cplx_t<R>;
  using P = PipeCfg<R, MM>;
  constexpr int K = P::K, H2 = P::H, HS = P::HS, PR = P::PR, NB = P::NB, S = P::S;
  constexpr int KP = (K + 1) / 2;
  constexpr int FA = 16 / (int)sizeof(C);  // samples per 16 bytes
  constexpr int NW = P::THREADS / 32;
  // a node's factors for this thread's halo row (a, b): the leading-dim
  // factors at halo cells a and b, and its K last-dim factors
  // hs = the node's stencil starts (h0, h1) in halo cells, loaded one node
  // ahead in the walks below (sten3 rows index the factors from them)
  // sten3 rows: stencil offset (h - start) clamped onto the block's zero;
  // halo-indexed rows: the factor at the halo cell itself
  auto fa = [&](const typename P::W* w, int2 hs, int a) {
    if constexpr (P::STEN3) return w[sten3_ow0(K) + min((unsigned)(a - hs.x), (unsigned)K)];
    else return w[a];
  };
  auto fb = [&](const typename P::W* w, int2 hs, int b) {
    if constexpr (P::STEN3) return w[sten3_ow1(K) + min((unsigned)(b - hs.y), (unsigned)K)];
    else return w[H2 + b];
  };
  constexpr int OWL = P::STEN3 ? STEN3_OW2 : 2 * H2;
  auto starts = [&](const int4* r) { return *reinterpret_cast<const int2*>(r); };
  extern __shared__ __align__(128) unsigned char smem[];
  // layout: ring stages | full[S] empty[S] meta[S] producer state | halo rows
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + P::CTL);
  unsigned long long* empty = full + S;
  StageMeta* meta = reinterpret_cast<StageMeta*>(empty + S);
  int* pst = reinterpret_cast<int*>(meta + S);  // producer: s, base, end, tile, k, last batch: nodes, slot
  C* stage = reinterpret_cast<C*>(smem + P::ROWS_OFF);  // per-thread staging rows
  const int lane = threadIdx.x & 31;
  static_assert(NB <= 32, "gather: one sample per lane of warp 0");
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full + i, GATHER ? 33 : 1);
      mbar_init(empty + i, NW);
    }
    pst[0] = blockIdx.x;
    pst[4] = 0;
    if (blockIdx.x < nsubs) {
      const int4 sp = subs[blockIdx.x];
      pst[1] = sp.y;
      pst[2] = sp.y + sp.z;
      pst[3] = sp.x;
    }
  }
  __syncthreads();

  // ---- producer (thread 0): state in shared memory, so thread 0 keeps no
  // extra registers live across the node loop
  auto produce = [&]() {
    const int pk = pst[4];
    const int slot = pk % S;
    if (pk >= S) mbar_wait(empty + slot, ((pk / S) - 1) & 1);
    StageMeta* mt = meta + slot;
    pst[4] = pk + 1;
    if (GATHER) {
      pst[5] = 0;
      pst[6] = slot;
    }
    if (pst[0] >= nsubs) {
      mt->nb = -1;
      mbar_arrive(full + slot);
      return;
    }
    const int pbase = pst[1], pend = pst[2];
    const int nb = min(NB, pend - pbase);
    const int foff = GATHER ? 0 : pbase & (FA - 1);
    const int fcnt = (nb + foff + FA - 1) & ~(FA - 1);
    mt->tile = pst[3];
    mt->nb = nb;
    mt->last = pbase + nb >= pend;
    mt->foff = foff;
    unsigned char* st = smem + slot * P::SB;
    const unsigned wb = (unsigned)(sizeof(typename P::W) * PR) * nb, rb = 16u * nb,
                   fb = GATHER ? 0u : (unsigned)sizeof(C) * fcnt;
    mbar_expect_tx(full + slot, wb + rb + fb);
    if (GATHER) pst[5] = nb;
    bulk_g2s(st, reinterpret_cast<const typename P::W*>(psi) + (int64_t)pbase * PR, wb, full + slot);
    bulk_g2s(st + P::W_BYTES, rec + pbase, rb, full + slot);
    if (!GATHER) bulk_g2s(st + P::W_BYTES + P::R_BYTES, fsorted + (pbase - foff), fb, full + slot);
    if (pbase + nb < pend) {
      pst[1] = pbase + nb;
    } else {
      const int s = next_sub(g, SCHED_SPREAD3, pst[0]);
      pst[0] = s;
      if (s < nsubs) {
        const int4 sp = subs[s];
        pst[1] = sp.y;
        pst[2] = sp.y + sp.z;
        pst[3] = sp.x;
      }
    }
  };
  auto fetch_idx = [&]() -> int {  // warp 0: this lane's sample index in the batch the producer points at
    const int b = pst[1] + lane;
    return pst[0] < nsubs && lane < NB && b < pst[2] ? perm[b] : 0;
  };
  int pidx = 0;
  const unsigned long long gpol = l2_evict_first_policy();
  auto produce_w = [&]() {  // warp 0, converged
    __syncwarp();
    if (lane == 0) produce();
    __syncwarp();
    const int slot = pst[6];
    if (lane < pst[5])
      cp_async_cell_hint<C>(reinterpret_cast<C*>(smem + slot * P::SB + P::W_BYTES + P::R_BYTES) + lane, funs + pidx,
                            gpol);
    cp_async_arrive_noinc(full + slot);
    pidx = fetch_idx();
  };
  if constexpr (GATHER) {
    if (threadIdx.x < 32) {
      pidx = fetch_idx();
      for (int i = 0; i < S - 1; ++i) produce_w();
    }
  } else {
    if (threadIdx.x == 0)
      for (int i = 0; i < S - 1; ++i) produce();
  }

  // contiguous row ownership: a warp holds ~1.5 halo a-lines and skips
  // (warp-uniformly) the nodes whose stencil misses them -- measured 12%
  // faster than strided ownership, where every warp sees every node.
  // Non-owners get an out-of-range row so the stencil test never passes.
  int k = 0;
  if constexpr (P::RUNACC) {
  // Run accumulators: the K cells a run of equal last-dim start touches stay
  // in registers (static indices, no switch); when the run start moves they
  // go to this thread's own shared-memory rows (no other thread touches
  // them: no atomics, no conflicts).  A thread owns RPT rows (a, b0 + j) of
  // one a-line, so one set of factor loads feeds RPT rows and fewer warps
  // walk each node.  [lo_w, hi_w) is the written part of the rows; cells
  // outside it are stored instead of added, so the rows need no zeroing, and
  // only the written part is bulk-reduced at the end of a tile.
  constexpr int RPT = P::RPT, HB = P::HB;
  const int grp = threadIdx.x;
  const bool gown = grp < P::GROUPS;  // padding threads own no row
  // staging rows stay with the thread (its own bulk reductions guard them)
  C* const myrow = stage + (size_t)(gown ? grp : 0) * RPT * HS;  // row j at myrow + j * HS
#ifdef NFFTK_RUNACC_ALT
  // alternating row maps (as in the whole-row path below): on odd tiles a
  // thread holds row group (grp + GROUPS/2) mod GROUPS, so a warp that owns
  // centre a-lines on one tile owns edge lines on the next
  constexpr int SHG = P::GROUPS / 2;
#else
  constexpr int SHG = 0;
#endif
  int tpar = 0;
  for (;;) {  // tiles of this CTA
    const int shift = tpar ? SHG : 0;
    tpar ^= 1;
    const int g2 = gown ? (grp + shift) % P::GROUPS : 0;
    const int a = g2 / HB, b0 = (g2 % HB) * RPT;
    auto owns = [&](int j) { return gown && b0 + j < H2; };
    // this warp's a-lines: one interval, or two when its groups wrap
    const int w0g = min((int)(threadIdx.x & ~31u), P::GROUPS - 1);
    const int w1g = min((int)(threadIdx.x | 31u), P::GROUPS - 1);
    const int s0g = (w0g + shift) % P::GROUPS, s1g = (w1g + shift) % P::GROUPS;
    const int wa_lo = s0g / HB, wa_hi = s0g <= s1g ? s1g / HB : H2 - 1;
    const int wb_lo = s0g <= s1g ? (1 << 20) : 0, wb_hi = s0g <= s1g ? -1 : s1g / HB;
    R accr[RPT][K], acci[RPT][K];
#pragma unroll
    for (int j = 0; j < RPT; ++j)
#pragma unroll
      for (int c = 0; c < K; ++c) accr[j][c] = acci[j][c] = 0;
    int lo_w = 0, hi_w = 0, cur_h = -1;
    bool run_touched = false, first_run = true;
    int tile = -1;
    // add register cells [0, CNT) of the window into row cells [cur_h, cur_h + CNT)
    auto flush_cells = [&](auto cnt_tag) {
      constexpr int CNT = decltype(cnt_tag)::value;
      if (first_run) {  // the previous tile's reduction has finished reading the rows
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        first_run = false;
        lo_w = hi_w = cur_h;
      }
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        if (!owns(j)) continue;
        C* rw = myrow + j * HS;
        for (int c = hi_w; c < cur_h; ++c) rw[c] = C{0, 0};
        for (int c = cur_h + CNT; c < lo_w; ++c) rw[c] = C{0, 0};
#pragma unroll
        for (int t = 0; t < CNT; ++t) {
          const int c = cur_h + t;
          C v = C{0, 0};
          if (c >= lo_w && c < hi_w) v = rw[c];
          v.x += accr[j][t];
          v.y += acci[j][t];
          rw[c] = v;
        }
      }
      lo_w = min(lo_w, cur_h);
      hi_w = max(hi_w, cur_h + CNT);
    };
    // the window moves to start h: by one cell, the leaving cell goes to the
    // rows and the registers slide; otherwise the whole window is flushed
    auto move_window = [&](int h) {
      if (run_touched && gown) {
        if (h == cur_h + 1 && h <= H2 - K) {
          flush_cells(std::integral_constant<int, 1>{});
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
#pragma unroll
            for (int t = 0; t + 1 < K; ++t) {
              accr[j][t] = accr[j][t + 1];
              acci[j][t] = acci[j][t + 1];
            }
            accr[j][K - 1] = acci[j][K - 1] = 0;
          }
        } else {
          flush_cells(std::integral_constant<int, K>{});
#pragma unroll
          for (int j = 0; j < RPT; ++j)
#pragma unroll
            for (int t = 0; t < K; ++t) accr[j][t] = acci[j][t] = 0;
          run_touched = false;
        }
      }
      cur_h = h;
    };
    for (;; ++k) {  // batches of the tile
      const int slot = k % S;
      mbar_wait(full + slot, (k / S) & 1);
      const StageMeta mt = meta[slot];
      if (mt.nb < 0) break;
      tile = mt.tile;
      const unsigned char* st = smem + slot * P::SB;
      const typename P::W* pw = reinterpret_cast<const typename P::W*>(st);
      const int4* pr = reinterpret_cast<const int4*>(st + P::W_BYTES);
      const C* pf = reinterpret_cast<const C*>(st + P::W_BYTES + P::R_BYTES) + mt.foff;
      const int nb = (g.debug & 2) ? 0 : mt.nb;
      auto hits = [&](const int4 r) {
        const int w0 = (int)((unsigned)r.w & 0xffu);
        return (unsigned)r.z <= (unsigned)(H2 - K) &&
               ((r.x <= wa_hi && r.x + w0 > wa_lo) || (r.x <= wb_hi && r.x + w0 > wb_lo));
      };
      // one node: coefficients f * w0[a] * w1[b0 + j] against the K last-dim factors
      auto node1 = [&](const typename P::W* w, int2 hs, const C* fp) {
        const typename P::W wa = fa(w, hs, a);
        R s[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) s[j] = (R)(wa * fb(w, hs, b0 + j));
        run_touched = true;
        const C f = *fp;
        const C* w2 = reinterpret_cast<const C*>(w + OWL);
        C v[KP];
#pragma unroll
        for (int p = 0; p < KP; ++p) v[p] = w2[p];
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          const R cr = f.x * s[j], ci = f.y * s[j];
#pragma unroll
          for (int p = 0; p < KP; ++p) {
            accr[j][2 * p] = fma(cr, (R)v[p].x, accr[j][2 * p]);
            acci[j][2 * p] = fma(ci, (R)v[p].x, acci[j][2 * p]);
            if (2 * p + 1 < K) {
              accr[j][2 * p + 1] = fma(cr, (R)v[p].y, accr[j][2 * p + 1]);
              acci[j][2 * p + 1] = fma(ci, (R)v[p].y, acci[j][2 * p + 1]);
            }
          }
        }
      };
      // this warp's nodes of the batch, run by run (see the whole-row path)
      static_assert(P::NB <= 32, "one ballot per batch");
      const int4 rl = lane < nb ? pr[lane] : make_int4(0, 0, -1, 0);
      unsigned mask = __ballot_sync(~0u, lane < nb && hits(rl));
      const int zup = __shfl_up_sync(~0u, rl.z, 1);
      const unsigned rstart = __ballot_sync(~0u, lane == 0 || rl.z != zup);
      while (mask) {
        const int j0 = __ffs(mask) - 1;
        const int h = __shfl_sync(~0u, rl.z, j0);
        const unsigned later = rstart & ~((2u << j0) - 1u);
        unsigned run = later ? mask & ((later & (0u - later)) - 1u) : mask;
        mask &= ~run;
        if (h != cur_h) move_window(h);
        // the next node's stencil starts are loaded under this node's FMAs
        int jj = __ffs(run) - 1;
        int2 hs = starts(pr + jj);
        for (;;) {
          run &= run - 1;
          const int jn = run ? __ffs(run) - 1 : jj;
          const int2 hn = starts(pr + jn);
          node1(pw + jj * PR, hs, pf + jj);
          if (!run) break;
          jj = jn;
          hs = hn;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
      if constexpr (GATHER) {
        if (threadIdx.x < 32) produce_w();
      } else {
        if (threadIdx.x == 0) produce();
      }
      if (mt.last) {
        ++k;
        break;
      }
    }
    if (tile < 0) break;  // end of work
    if (run_touched && gown) flush_cells(std::integral_constant<int, K>{});
    if (gown && !first_run && !(g.debug & 1)) {
      int lo = lo_w, hi = hi_w;
      int tc[3];
      tile_of<3>(g, tile, tc);
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        if (!owns(j)) continue;
        C* rw = myrow + j * HS;
        if constexpr (sizeof(R) == 4) {  // c64: 16-byte pieces (m, n even: spread_dense_ok)
          if (lo & 1) rw[lo - 1] = C{0, 0};
          if (hi & 1) rw[hi] = C{0, 0};
        }
      }
      if constexpr (sizeof(R) == 4) {
        lo -= lo & 1;
        hi += hi & 1;
      }
      fence_proxy_async_smem();
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        if (!owns(j)) continue;
        const int b = b0 + j;
        C* rw = myrow + j * HS;
        if (g.dense_flush) {
          int ad = tc[0] * 8 + a - g.m, bd = tc[1] * 8 + b - g.m;
          ad += ad < 0 ? g.n[0] : (ad >= g.n[0] ? -g.n[0] : 0);
          bd += bd < 0 ? g.n[1] : (bd >= g.n[1] ? -g.n[1] : 0);
          int c0 = tc[2] * 8 - g.m + lo;
          c0 -= c0 >= g.n[2] ? g.n[2] : 0;
          bulk_red_row_wrapped<R>(gp, ((int64_t)ad * g.n[1] + bd) * g.n[2], c0, g.n[2], rw + lo, hi - lo);
        } else {
          int64_t row0 = ((int64_t)(tc[0] * 8 + a) * g.np[1] + tc[1] * 8 + b) * g.np[2] + tc[2] * 8 + lo;
          bulk_red_add<R>(gp + row0, rw + lo, (unsigned)((hi - lo) * sizeof(C)));
        }
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::);
    }
  }
  } else {
  const int row = threadIdx.x;       // also this thread's staging slot
  const bool owner = row < P::ROWS;  // non-owners accumulate garbage that is never flushed
#ifdef NFFTK_NO_ALT_ROWS
  constexpr int SH = 0;
#else
  // Alternating row maps: on odd tiles a thread holds halo row (row + SH) mod
  // ROWS, about half a halo further on, so a warp that owns well-covered
  // centre a-lines on one tile owns thinly covered edge lines on the next.
  // The node ring (S - 1 stages ahead) lets fast warps run into the next
  // tile, so over a pair of tiles every warp does about the same work
  // instead of the centre warps setting the pace of every tile.
  constexpr int SH = P::ROWS / 2;
#endif
  int tpar = 0;
  for (;;) {  // tiles of this CTA
    const int shift = tpar ? SH : 0;
    tpar ^= 1;
    const int rr = owner ? (row + shift) % P::ROWS : 0;
    const int a = rr / H2, b = rr % H2;
    // this warp's a-lines: one interval, or two when its rows wrap
    const int w0 = (int)(threadIdx.x & ~31u), w1 = min((int)(threadIdx.x | 31u), P::ROWS - 1);
    const int s0 = (w0 + shift) % P::ROWS, s1 = (w1 + shift) % P::ROWS;
    const int wa_lo = s0 / H2, wa_hi = s0 <= s1 ? s1 / H2 : H2 - 1;
    const int wb_lo = s0 <= s1 ? (1 << 20) : 0, wb_hi = s0 <= s1 ? -1 : s1 / H2;
    R accr[H2], acci[H2];
#pragma unroll
    for (int c = 0; c < H2; ++c) accr[c] = acci[c] = 0;
    bool touched = false;
    int tile = -1;
    for (;; ++k) {  // batches of the tile
      const int slot = k % S;
      mbar_wait(full + slot, (k / S) & 1);
      const StageMeta mt = meta[slot];
      if (mt.nb < 0) break;
      tile = mt.tile;
      const unsigned char* st = smem + slot * P::SB;
      const typename P::W* ws = reinterpret_cast<const typename P::W*>(st);
      const int4* rs = reinterpret_cast<const int4*>(st + P::W_BYTES);
      const C* fv = reinterpret_cast<const C*>(st + P::W_BYTES + P::R_BYTES) + mt.foff;
      const int nb = (g.debug & 2) ? 0 : mt.nb;
      // Per-batch warp view: lane l holds node l's record; one ballot gives
      // the nodes whose stencil meets this warp's rows, another the run
      // starts (last-dim start changes).  The walk then visits only this
      // warp's nodes, run by run, with bit operations between nodes -- no
      // record load or test on the node-to-node path.
      static_assert(P::NB <= 32, "one ballot per batch");
      const int4 rl = lane < nb ? rs[lane] : make_int4(0, 0, -1, 0);
      const int rw0 = (int)((unsigned)rl.w & 0xffu);
      unsigned mask = __ballot_sync(~0u, lane < nb && (unsigned)rl.z <= (unsigned)(H2 - K) &&
                                              ((rl.x <= wa_hi && rl.x + rw0 > wa_lo) ||
                                               (rl.x <= wb_hi && rl.x + rw0 > wb_lo)));
      const int zup = __shfl_up_sync(~0u, rl.z, 1);
      const unsigned rstart = __ballot_sync(~0u, lane == 0 || rl.z != zup);
      while (mask) {
        const int j0 = __ffs(mask) - 1;
        const int h = __shfl_sync(~0u, rl.z, j0);
        const unsigned later = rstart & ~((2u << j0) - 1u);  // run starts after j0 (2u << 31 == 0)
        const unsigned run = later ? mask & ((later & (0u - later)) - 1u) : mask;
        mask &= ~run;
        touched = true;
#define NFFTK_PIPE_NODE(H)                                                                 \
  {                                                                                        \
    m2 &= m2 - 1;                                                                          \
    const int jn = m2 ? __ffs(m2) - 1 : jj;                                                \
    const int2 hn = starts(rs + jn); /* next node's starts, under this node's FMAs */      \
    const typename P::W* pw = ws + jj * PR;                                                \
    const R s = (R)(fa(pw, hs, a) * fb(pw, hs, b));                                        \
    const C f = fv[jj];                                                                    \
    const R cr = f.x * s, ci = f.y * s;                                                    \
    const C* w2 = reinterpret_cast<const C*>(pw + OWL); /* factor pairs */                 \
    _Pragma("unroll") for (int p = 0; p < KP; ++p) {                                       \
      const C v = w2[p];                                                                   \
      accr[H + 2 * p] = fma(cr, (R)v.x, accr[H + 2 * p]);                                  \
      acci[H + 2 * p] = fma(ci, (R)v.x, acci[H + 2 * p]);                                  \
      if (2 * p + 1 < K) {                                                                 \
        accr[H + 2 * p + 1] = fma(cr, (R)v.y, accr[H + 2 * p + 1]);                        \
        acci[H + 2 * p + 1] = fma(ci, (R)v.y, acci[H + 2 * p + 1]);                        \
      }                                                                                    \
    }                                                                                      \
    jj = jn;                                                                               \
    hs = hn;                                                                               \
  }
#define NFFTK_PIPE_CASE(H)                                                     \
  case H:                                                                      \
    if constexpr (H + K <= H2) {                                               \
      unsigned m2 = run;                                                       \
      int jj = __ffs(m2) - 1;                                                  \
      int2 hs = starts(rs + jj);                                               \
      do {                                                                     \
        NFFTK_PIPE_NODE(H)                                                     \
      } while (m2);                                                            \
    }                                                                          \
    break;
        switch (h) {
          NFFTK_PIPE_CASE(0) NFFTK_PIPE_CASE(1) NFFTK_PIPE_CASE(2) NFFTK_PIPE_CASE(3)
          NFFTK_PIPE_CASE(4) NFFTK_PIPE_CASE(5) NFFTK_PIPE_CASE(6) NFFTK_PIPE_CASE(7)
          NFFTK_PIPE_CASE(8)
          default:
            break;
        }
#undef NFFTK_PIPE_CASE
#undef NFFTK_PIPE_NODE
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
      if constexpr (GATHER) {
        if (threadIdx.x < 32) produce_w();
      } else {
        if (threadIdx.x == 0) produce();
      }
      if (mt.last) {
        ++k;
        break;
      }
    }
    if (tile < 0) break;  // end of work
    // tile done: each thread stages and bulk-reduces its own row -- no CTA
    // barrier; the row slot is reused only after this thread's previous
    // reduction finished reading it
    if (owner && touched && !(g.debug & 1)) {
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      C* dst = stage + (size_t)row * HS;
#pragma unroll
      for (int c = 0; c < H2; ++c) {
        C v;
        v.x = accr[c];
        v.y = acci[c];
        dst[c] = v;
      }
      if constexpr (HS > H2) {
        C z;
        z.x = 0;
        z.y = 0;
        dst[H2] = z;
      }
      fence_proxy_async_smem();
      int tc[3];
      tile_of<3>(g, tile, tc);
      if (g.dense_flush) {
        // halo cell (a, b, c) of the tile is dense slot tile * T + (a, b, c) - m;
        // the row goes out as HS cells (c64: one trailing zero keeps 16 bytes)
        int ad = tc[0] * 8 + a - g.m, bd = tc[1] * 8 + b - g.m;
        ad += ad < 0 ? g.n[0] : (ad >= g.n[0] ? -g.n[0] : 0);
        bd += bd < 0 ? g.n[1] : (bd >= g.n[1] ? -g.n[1] : 0);
        bulk_red_row_wrapped<R>(gp, ((int64_t)ad * g.n[1] + bd) * g.n[2], tc[2] * 8 - g.m, g.n[2], dst, HS);
        asm volatile("cp.async.bulk.commit_group;\n" ::);
        continue;
      }
      int64_t row0 = ((int64_t)(tc[0] * 8 + a) * g.np[1] + tc[1] * 8 + b) * g.np[2] + tc[2] * 8;
      bulk_red_add<R>(gp + row0, dst, (unsigned)(HS * sizeof(C)));
      asm volatile("cp.async.bulk.commit_group;\n" ::);
    }
  }
  }  // RUNACC
  if (threadIdx.x == 0) sched_done(g, SCHED_SPREAD3);
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

// ------------------------------------- C'': pipelined register spread, d = 2
// One warp per CTA, one 32-row halo per tile: lane l owns halo row a = l
// (T0 = 32 - (2m+1)) and keeps its H1 = T1 + 2m + 1 cells in registers.  A
// node is 2m+1 FMA pairs on the lanes inside its row window; batches arrive
// on the same TMA/mbarrier ring as the d = 3 kernel (lane 0 produces, lag 1),
// nodes come in runs of equal last-dim stencil start, and each lane
// bulk-reduces its own row at the end of a tile.
template <typename R, int MM, int T1>
struct Pipe2Cfg {
  static constexpr int K = 2 * MM + 1;
  static constexpr int H0 = 32;
  static constexpr int H1 = T1 + K;
  static constexpr int ELEM = 2 * (int)sizeof(R);
  static constexpr int HS = ELEM == 8 ? H1 + (H1 & 1) : H1;  // 16-byte rows
  using W = R;                                                // factor type (fp32 rows for c64)
  static constexpr int PR = psi_row_pad<W>(2 * K);            // stencil-indexed PRE_PSI row
  static constexpr int NB = 16;
  // ring depth: measured at C4 (A/B, tools/ab_c4.sh) -- 3 stages for fp32
  // (spread 1.85 -> 1.71 ms: smaller CTAs, more of them per SM), 4 for fp64
  // (3 stages: 2.86 -> 3.29 ms)
  static constexpr int S = sizeof(R) == 4 ? 3 : 4;
  static constexpr size_t al(size_t v) { return (v + 15) & ~(size_t)15; }
  static constexpr size_t W_BYTES = al(sizeof(W) * NB * PR);
  static constexpr size_t R_BYTES = al(16 * (size_t)NB);
  static constexpr size_t SB = W_BYTES + R_BYTES + al((size_t)ELEM * (NB + 2));
  static constexpr size_t CTL = S * SB;
  static constexpr size_t ROWS_OFF = CTL + al(16 * (size_t)S + sizeof(StageMeta) * S + 32);
  static constexpr size_t SMEM = ROWS_OFF + al((size_t)H0 * HS * ELEM);
};

// GATHER: the samples are not read from a sorted copy but fetched by warp 0
// itself, lane l < NB bringing f[perm[base + l]] of the batch with one
// cp.async that arrives on the batch's mbarrier (as in residue.cu).
// NWARP warps share a tile: warp w takes nodes w, w + NWARP, ... of every
// batch into its own register halo, and at the end of the tile the halos are
// added up in the staging rows (lane a of every warp owns row a: no
// conflicts) before one flush.  The ring and the staging rows -- the shared
// memory that limited the one-warp CTAs to 8 warps per SM at C4 -- serve
// NWARP warps; registers (84 accumulators per lane) stop it at two.
template <typename R, int MM, int T1, bool GATHER, int NWARP>
__global__ void __launch_bounds__(32 * NWARP)
k_spread2_pipe(cplx_t<R>* __restrict__ gp, const cplx_t<R>* __restrict__ fsorted,
               const cplx_t<R>* __restrict__ funs, const int* __restrict__ perm,
               const double* __restrict__ psi, const int4* __restrict__ rec,
               const int4* __restrict__ subs, int nsubs, Geom g) {
  using C = cplx_t<R>;
  using P = Pipe2Cfg<R, MM, T1>;
  constexpr int K = P::K, H1 = P::H1, HS = P::HS, PR = P::PR, NB = P::NB, S = P::S;
  constexpr int FA = 16 / (int)sizeof(C);
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + P::CTL);
  unsigned long long* empty = full + S;
  StageMeta* meta = reinterpret_cast<StageMeta*>(empty + S);
  int* pst = reinterpret_cast<int*>(meta + S);  // producer: s, base, end, tile, k, last batch: nodes, slot
  C* stage = reinterpret_cast<C*>(smem + P::ROWS_OFF);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full + i, GATHER ? 33 : 1);
      mbar_init(empty + i, NWARP);
    }
    pst[0] = blockIdx.x;
    pst[4] = 0;
    if (blockIdx.x < nsubs) {
      const int4 sp = subs[blockIdx.x];
      pst[1] = sp.y;
      pst[2] = sp.y + sp.z;
      pst[3] = sp.x;
    }
  }
  if constexpr (NWARP > 1) __syncthreads();
  else __syncwarp();
  auto produce = [&]() {
    const int pk = pst[4];
    const int slot = pk % S;
    if (pk >= S) mbar_wait(empty + slot, ((pk / S) - 1) & 1);
    StageMeta* mt = meta + slot;
    pst[4] = pk + 1;
    if (GATHER) {
      pst[5] = 0;
      pst[6] = slot;
    }
    if (pst[0] >= nsubs) {
      mt->nb = -1;
      mbar_arrive(full + slot);
      return;
    }
    const int pbase = pst[1], pend = pst[2];
    const int nb = min(NB, pend - pbase);
    const int foff = pbase & (FA - 1);
    const int fcnt = (nb + foff + FA - 1) & ~(FA - 1);
    mt->tile = pst[3];
    mt->nb = nb;
    mt->last = pbase + nb >= pend;
    mt->foff = foff;
    unsigned char* st = smem + slot * P::SB;
    const unsigned wb = (unsigned)(sizeof(typename P::W) * PR) * nb, rb = 16u * nb,
                   fb = GATHER ? 0u : (unsigned)sizeof(C) * fcnt;
    mbar_expect_tx(full + slot, wb + rb + fb);
    if (GATHER) pst[5] = nb;
    bulk_g2s(st, reinterpret_cast<const typename P::W*>(psi) + (int64_t)pbase * PR, wb, full + slot);
    bulk_g2s(st + P::W_BYTES, rec + pbase, rb, full + slot);
    if (!GATHER) bulk_g2s(st + P::W_BYTES + P::R_BYTES, fsorted + (pbase - foff), fb, full + slot);
    if (pbase + nb < pend) {
      pst[1] = pbase + nb;
    } else {
      const int s = next_sub(g, SCHED_SPREAD2, pst[0]);
      pst[0] = s;
      if (s < nsubs) {
        const int4 sp = subs[s];
        pst[1] = sp.y;
        pst[2] = sp.y + sp.z;
        pst[3] = sp.x;
      }
    }
  };
  // index of this lane's sample in the batch the producer state points at
  auto fetch_idx = [&]() -> int {
    const int b = pst[1] + lane;
    return pst[0] < nsubs && lane < NB && b < pst[2] ? perm[b] : 0;
  };
  int pidx = 0;
  auto produce_w = [&]() {  // the whole warp, converged
    __syncwarp();
    if (lane == 0) produce();
    __syncwarp();
    const int slot = pst[6];
    if (lane < pst[5])
      cp_async_cell<C>(reinterpret_cast<C*>(smem + slot * P::SB + P::W_BYTES + P::R_BYTES) + lane, funs + pidx);
    cp_async_arrive_noinc(full + slot);
    pidx = fetch_idx();
  };
  if (warp == 0) {
    if constexpr (GATHER) {
      pidx = fetch_idx();
      for (int i = 0; i < S - 1; ++i) produce_w();
    } else {
      if (lane == 0)
        for (int i = 0; i < S - 1; ++i) produce();
    }
  }
  __syncwarp();

  const int a = lane;
  int k = 0;
  for (;;) {  // tiles of this CTA
    R accr[H1], acci[H1];
#pragma unroll
    for (int c = 0; c < H1; ++c) accr[c] = acci[c] = 0;
    int tile = -1;
    for (;; ++k) {  // batches of the tile
      const int slot = k % S;
      mbar_wait(full + slot, (k / S) & 1);
      const StageMeta mt = meta[slot];
      if (mt.nb < 0) break;
      tile = mt.tile;
      const unsigned char* st = smem + slot * P::SB;
      const typename P::W* ws = reinterpret_cast<const typename P::W*>(st);
      const int4* rs = reinterpret_cast<const int4*>(st + P::W_BYTES);
      const C* fv = reinterpret_cast<const C*>(st + P::W_BYTES + P::R_BYTES) + (GATHER ? 0 : mt.foff);
      const int nb = (g.debug & 2) ? 0 : mt.nb;
      int jb = warp;  // this warp's nodes: warp, warp + NWARP, ...
      int4 r = jb < nb ? rs[jb] : make_int4(0, 0, 0, 0);
      while (jb < nb) {
#define NFFTK_PIPE2_NODE(H)                                                                \
  {                                                                                        \
    const int ta = a - r.x;                                                                \
    const bool act = (unsigned)ta < ((unsigned)r.w & 0xffu);                               \
    const typename P::W* w = ws + jb * PR;                                                 \
    const typename P::W s0 = w[min((unsigned)ta, (unsigned)(K - 1))];                      \
    const R s = act ? (R)s0 : (R)0;                                                        \
    const C f = fv[jb];                                                                    \
    const R cr = f.x * s, ci = f.y * s;                                                    \
    const typename P::W* w1 = w + K;                                                       \
    _Pragma("unroll") for (int t = 0; t < K; ++t) {                                        \
      accr[H + t] = fma(cr, (R)w1[t], accr[H + t]);                                        \
      acci[H + t] = fma(ci, (R)w1[t], acci[H + t]);                                        \
    }                                                                                      \
  }
#define NFFTK_PIPE2_CASE(H)                                  \
  case H:                                                    \
    if constexpr (H + K <= H1) {                             \
      for (;;) {                                             \
        NFFTK_PIPE2_NODE(H)                                  \
        if ((jb += NWARP) >= nb) break;                      \
        r = rs[jb];                                          \
        if (r.y != H) break;                                 \
      }                                                      \
    } else {                                                 \
      if ((jb += NWARP) < nb) r = rs[jb];                    \
    }                                                        \
    break;
        switch (r.y) {
          NFFTK_PIPE2_CASE(0) NFFTK_PIPE2_CASE(1) NFFTK_PIPE2_CASE(2) NFFTK_PIPE2_CASE(3)
          NFFTK_PIPE2_CASE(4) NFFTK_PIPE2_CASE(5) NFFTK_PIPE2_CASE(6) NFFTK_PIPE2_CASE(7)
          NFFTK_PIPE2_CASE(8) NFFTK_PIPE2_CASE(9) NFFTK_PIPE2_CASE(10) NFFTK_PIPE2_CASE(11)
          NFFTK_PIPE2_CASE(12) NFFTK_PIPE2_CASE(13) NFFTK_PIPE2_CASE(14) NFFTK_PIPE2_CASE(15)
          NFFTK_PIPE2_CASE(16)
          default:
            if ((jb += NWARP) < nb) r = rs[jb];
            break;
        }
#undef NFFTK_PIPE2_CASE
#undef NFFTK_PIPE2_NODE
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
      if (warp == 0) {
        if constexpr (GATHER) produce_w();
        else if (lane == 0) produce();
      }
      __syncwarp();
      if (mt.last) {
        ++k;
        break;
      }
    }
    if (tile < 0) break;  // end of work
    if (!(g.debug & 1)) {
      // warp 0 stages its rows once the previous flush has read the staging
      // area, the other warps add theirs, warp 0 sends the sums
      C* dst = stage + (size_t)a * HS;
      if (warp == 0) {
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
#pragma unroll
        for (int c = 0; c < H1; ++c) {
          C v;
          v.x = accr[c];
          v.y = acci[c];
          dst[c] = v;
        }
        if constexpr (HS > H1) {
          C z;
          z.x = 0;
          z.y = 0;
          dst[H1] = z;
        }
      }
#pragma unroll
      for (int w = 1; w < NWARP; ++w) {
        __syncthreads();
        if (warp == w) {
#pragma unroll
          for (int c = 0; c < H1; ++c) {
            C v = dst[c];
            v.x += accr[c];
            v.y += acci[c];
            dst[c] = v;
          }
        }
      }
      if constexpr (NWARP > 1) __syncthreads();
      if (warp == 0) {
        fence_proxy_async_smem();
        const int t0 = tile / g.ntile[1], t1 = tile - t0 * g.ntile[1];
        bool done = false;
        if (g.dense_flush) {
          int ad = t0 * g.T[0] + a - g.m;
          ad += ad < 0 ? g.n[0] : (ad >= g.n[0] ? -g.n[0] : 0);
          bulk_red_row_wrapped<R>(gp, (int64_t)ad * g.n[1], t1 * T1 - g.m, g.n[1], dst, HS);
          done = true;
        }
        if (!done) {
          int64_t row0 = (int64_t)(t0 * g.T[0] + a) * g.np[1] + t1 * T1;
          bulk_red_add<R>(gp + row0, dst, (unsigned)(HS * sizeof(C)));
        }
        asm volatile("cp.async.bulk.commit_group;\n" ::);
      }
    }
  }
  if (threadIdx.x == 0) sched_done(g, SCHED_SPREAD2);
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

bool spread2_pipe_ok(const Geom& g) {
  return g.d == 2 && g.mode == MODE_TENSOR && g.psi && g.rec && pipe_geometry(g);
}

// Spreads that fetch their samples through perm themselves (no sorted copy,
// no k_permute_samples): the residue spread and the pipelined d = 2 / d = 3 ones.
bool spread_pipe_ok(const Geom& g, int elem_bytes);
bool spread_gathers(const Geom& g, bool single) {
  if (getenv("NFFTK_NO_GATHER")) return false;
  if (res_ok(g)) return res_gathers(g, single);
  return spread2_pipe_ok(g) || (g.d == 3 && g.m <= 6 && spread_pipe_ok(g, single ? 8 : 16));
}

bool spread_pipe_ok(const Geom& g, int elem_bytes) {
  (void)elem_bytes;
  return g.d == 3 && g.mode == MODE_TENSOR && g.psi && g.rec && g.psi_pad;
}

// The pipelined c128 spreads can reduce straight into the dense grid (rows
// wrapped periodically, bulk_red_row_wrapped) instead of the ghost-padded
// grid + fold: every halo row must fit in one period (H <= n).
bool spread_dense_ok(const Geom& g, int elem_bytes) {
  if (getenv("NFFTK_NO_DENSE_FLUSH")) return false;
  // c64: 8-byte cells, so the row start (tile * 8 - m), the staged row (HS,
  // even) and the period must all be even to keep 16-byte bulk reductions
  if (elem_bytes == 8 && (g.m % 2 != 0 || g.n[g.d - 1] % 2 != 0 || g.HS % 2 != 0)) return false;
  const bool pipe = (g.d == 3 && g.m <= 6 && spread_pipe_ok(g, elem_bytes)) || (g.d == 2 && spread2_pipe_ok(g));
  if (!pipe) return false;
  for (int i = 0; i < g.d; ++i)
    if (g.H[i] > g.n[i]) return false;
  return g.HS <= g.n[g.d - 1];
}

size_t spread_rr_smem(const Geom& g, int elem_bytes) {
  const int K = 2 * g.m + 1;
  auto al = [](size_t v) { return (v + 15) & ~(size_t)15; };
  size_t rows = (size_t)g.H[0] * g.H[1];
  return al(rows * g.HS * elem_bytes) + al((size_t)g.nb_spread * K * elem_bytes) +
         2 * batch_bytes_of(3, g.nb_spread, K, elem_bytes);
}

// ================================================================ launchers
static size_t halo_bytes(const Geom& g, int elem_bytes) {
  size_t rows = 1;
  for (int i = 0; i < g.d - 1; ++i) rows *= g.H[i];
  return ((rows * g.HS * elem_bytes) + 15) & ~(size_t)15;
}

size_t interp_smem(const Geom& g, int elem_bytes, int threads) {
  (void)threads;
  return halo_bytes(g, elem_bytes) + 16 + 2 * batch_bytes_of(g.d, INTERP_NB, 2 * g.m + 1, elem_bytes);
}

size_t spread_smem_nb(const Geom& g, int elem_bytes, int nb) {
  const int K = 2 * g.m + 1, WF = 2 * g.m;
  auto al = [](size_t v) { return (v + 15) & ~(size_t)15; };
  size_t s = halo_bytes(g, elem_bytes) + al((size_t)nb * K * elem_bytes);
  if (g.d == 3) s += al((size_t)nb * WF * WF * sizeof(double));
  return s + 2 * batch_bytes_of(g.d, nb, K, elem_bytes);
}

size_t spread_smem(const Geom& g, int elem_bytes) { return spread_smem_nb(g, elem_bytes, g.nb_spread); }

int spread_threads(const Geom& g) {
  // d=3: one warp per owned a-row class (2m warps); d=1, 2: one warp
  if (g.d == 3) return 32 * std::max(2, std::min(16, 2 * g.m));
  return 32;
}

template <typename R, int D, int MM>
static void interp_go(const CUtensorMap* tm, const void* gp, void* f, void*, const double* xs,
                      const int* perm, const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  if constexpr (D >= 2 && MM > 0 && IPipeCfg<R, D, MM>::SMEM <= 224 * 1024) {
    if (interp_pipe_ok(g)) {
      using P = IPipeCfg<R, D, MM>;
      if (g.HS != P::HS) fail(EK_CUDA, "pipe interp: halo row stride mismatch");
      if (D == 3 && g.psi_pad != (P::STEN3 ? 2 : 1)) fail(EK_CUDA, "pipe interp: PRE_PSI layout mismatch");
      auto kern = k_interp_pipe<R, D, MM>;
      NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
      static int sms = 0;
      if (!sms) {
        int dev = 0;
        NFFTK_CUDA(cudaGetDevice(&dev));
        NFFTK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      }
      int per_sm = 0;
      NFFTK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, P::THREADS, P::SMEM));
      int grid = std::max(1, std::min(nsubs, sms * std::max(1, per_sm)));
      kern<<<grid, P::THREADS, P::SMEM, s>>>(*tm, (cplx_t<R>*)f, g.psi, g.rec, perm, subs, nsubs,
                                           sched_geom(g, nsubs, grid, 16));
      count_launch();
      return;
    }
  }
  const int threads = g.nt_interp;
  size_t smem = interp_smem(g, sizeof(cplx_t<R>), threads);
  auto kern = k_interp<R, D, MM>;
  NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<nsubs, threads, smem, s>>>(*tm, (const cplx_t<R>*)gp, (cplx_t<R>*)f, xs, perm, subs, g);
  count_launch();
}

bool spread_rr_ok(const Geom& g, int elem_bytes) {
  return g.d == 3 && g.m >= 1 && g.m <= 8 && g.T[0] == 8 && g.T[1] == 8 && g.T[2] == 8 &&
         g.H[0] * g.H[1] <= 512 &&
         spread_rr_smem(g, elem_bytes) <= 220 * 1024 && !getenv("NFFTK_NO_RR");
}

void launch_permute(bool single, const void* f, const int* perm, int64_t M, void* fs, cudaStream_t s) {
  unsigned blocks = (unsigned)std::min<int64_t>((M + 255) / 256, 148 * 64);
  if (single) k_permute_samples<float2><<<blocks, 256, 0, s>>>((const float2*)f, perm, M, (float2*)fs);
  else k_permute_samples<double2><<<blocks, 256, 0, s>>>((const double2*)f, perm, M, (double2*)fs);
  count_launch();
}

template <typename R, int D, int MM>
static void spread_go(const CUtensorMap*, void* gp, const void* f, void* fs, const double* xs,
                      const int* perm, const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  if constexpr (D == 3 && MM > 0) {
    if constexpr (MM <= 6) {
      if (spread_pipe_ok(g, sizeof(cplx_t<R>))) {
        using P = PipeCfg<R, MM>;
        static_assert(P::NB > 0 && P::S >= 2, "pipe ring does not fit");
        if (g.HS != P::HS) fail(EK_CUDA, "pipe spread: halo row stride mismatch");
        if (g.psi_pad != (P::STEN3 ? 2 : 1)) fail(EK_CUDA, "pipe spread: PRE_PSI layout mismatch");
        const bool gather = spread_gathers(g, sizeof(R) == 4);
        auto kern = gather ? k_spread_pipe<R, MM, true> : k_spread_pipe<R, MM, false>;
        NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
        static int sms = 0;
        if (!sms) {
          int dev = 0;
          NFFTK_CUDA(cudaGetDevice(&dev));
          NFFTK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        }
        int per_sm = 0;
        NFFTK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, P::THREADS, P::SMEM));
        int grid = std::max(1, std::min(nsubs, sms * std::max(1, per_sm)));
        kern<<<grid, P::THREADS, P::SMEM, s>>>((cplx_t<R>*)gp, (const cplx_t<R>*)fs, (const cplx_t<R>*)f,
                                               gather ? perm : nullptr, g.psi, g.rec, subs, nsubs,
                                               sched_geom(g, nsubs, grid));
        count_launch();
        return;
      }
    }
    if (spread_rr_ok(g, sizeof(cplx_t<R>))) {
      const int threads = (g.H[0] * g.H[1] + 31) & ~31;
      size_t smem = spread_rr_smem(g, sizeof(cplx_t<R>));
      auto kern = k_spread_rr<R, MM, 8>;
      NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      // persistent CTAs: as many as fit on the device at once
      static int sms = 0;
      if (!sms) {
        int dev = 0;
        NFFTK_CUDA(cudaGetDevice(&dev));
        NFFTK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      }
      int per_sm = 0;
      NFFTK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
      int grid = std::max(1, std::min(nsubs, sms * std::max(1, per_sm)));
      kern<<<grid, threads, smem, s>>>((cplx_t<R>*)gp, (const cplx_t<R>*)fs, xs, subs, nsubs, g);
      count_launch();
      return;
    }
  }
  if constexpr (D == 2 && MM > 0) {
    if (spread2_pipe_ok(g)) {
      using P = Pipe2Cfg<R, MM, 8>;
      if (g.HS != P::HS) fail(EK_CUDA, "pipe spread: halo row stride mismatch");
      const bool gather = spread_gathers(g, sizeof(R) == 4);
      // complex128: two warps per tile (C4 spread 2.32 -> 2.00 ms: twice the
      // warps on the same ring and staging rows); complex64 stays at one
      // (1.36 ms with one, 1.37 with two, 1.70 with four).  NFFTK_SPREAD2_WARPS
      // overrides for A/B runs and tests.
      const char* we = getenv("NFFTK_SPREAD2_WARPS");
      int nwarp = we ? atoi(we) : (sizeof(R) == 8 ? 2 : 1);
      if (nwarp != 1 && nwarp != 2) nwarp = 2;
      auto kern = gather ? k_spread2_pipe<R, MM, 8, true, 2> : k_spread2_pipe<R, MM, 8, false, 2>;
      if (nwarp == 1) kern = gather ? k_spread2_pipe<R, MM, 8, true, 1> : k_spread2_pipe<R, MM, 8, false, 1>;
      NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
      static int sms2 = 0;
      if (!sms2) {
        int dev = 0;
        NFFTK_CUDA(cudaGetDevice(&dev));
        NFFTK_CUDA(cudaDeviceGetAttribute(&sms2, cudaDevAttrMultiProcessorCount, dev));
      }
      int per_sm = 0;
      NFFTK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * nwarp, P::SMEM));
      int grid = std::max(1, std::min(nsubs, sms2 * std::max(1, per_sm)));
      kern<<<grid, 32 * nwarp, P::SMEM, s>>>((cplx_t<R>*)gp, (const cplx_t<R>*)fs, (const cplx_t<R>*)f,
                                     gather ? perm : nullptr, g.psi, g.rec, subs, nsubs,
                                     sched_geom(g, nsubs, grid));
      count_launch();
      return;
    }
  }
  const int threads = spread_threads(g);
  size_t smem = spread_smem(g, sizeof(cplx_t<R>));
  auto kern = k_spread<R, D, MM>;
  NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<nsubs, threads, smem, s>>>((cplx_t<R>*)gp, (const cplx_t<R>*)fs, xs, subs, g);
  count_launch();
}

#define NFFTK_DISPATCH_M(FN, R, D, ...)                      \
  switch (g.m) {                                             \
    case 1: FN<R, D, 1>(__VA_ARGS__); break;                 \
    case 2: FN<R, D, 2>(__VA_ARGS__); break;                 \
    case 3: FN<R, D, 3>(__VA_ARGS__); break;                 \
    case 4: FN<R, D, 4>(__VA_ARGS__); break;                 \
    case 5: FN<R, D, 5>(__VA_ARGS__); break;                 \
    case 6: FN<R, D, 6>(__VA_ARGS__); break;                 \
    case 7: FN<R, D, 7>(__VA_ARGS__); break;                 \
    case 8: FN<R, D, 8>(__VA_ARGS__); break;                 \
    default: FN<R, D, 0>(__VA_ARGS__); break;                \
  }

#define NFFTK_DISPATCH_DM(FN, R, ...)                                  \
  do {                                                                 \
    if (g.d == 1) { NFFTK_DISPATCH_M(FN, R, 1, __VA_ARGS__) }          \
    else if (g.d == 2) { NFFTK_DISPATCH_M(FN, R, 2, __VA_ARGS__) }     \
    else { NFFTK_DISPATCH_M(FN, R, 3, __VA_ARGS__) }                   \
  } while (0)

void launch_interp(bool single, const void* tmap, const void* gp, void* f, const double* xs,
                   const int* perm, const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  if (nsubs <= 0) return;
  const CUtensorMap* tm = (const CUtensorMap*)tmap;
  if (single) NFFTK_DISPATCH_DM(interp_go, float, tm, gp, f, nullptr, xs, perm, subs, nsubs, g, s);
  else NFFTK_DISPATCH_DM(interp_go, double, tm, gp, f, nullptr, xs, perm, subs, nsubs, g, s);
}

void launch_spread(bool single, void* gp, const void* f, void* fs, const double* xs,
                   const int* perm, const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  if (nsubs <= 0) return;
  if (res_ok(g)) {  // gp: the dense grid (dense_flush)
    launch_spread_res(single, gp, fs, f, perm, xs, subs, nsubs, g, s);
    return;
  }
  const CUtensorMap* tm = nullptr;
  if (single) NFFTK_DISPATCH_DM(spread_go, float, tm, gp, f, fs, xs, perm, subs, nsubs, g, s);
  else NFFTK_DISPATCH_DM(spread_go, double, tm, gp, f, fs, xs, perm, subs, nsubs, g, s);
}

}  // namespace nfftk
