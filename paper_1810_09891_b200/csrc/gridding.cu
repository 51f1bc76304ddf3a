// Gridding kernels of the nfftk hot path (sm_100a):
//   B   (interp) : f_j = sum_l g[l mod n] prod_i psi_i(x_ji - l_i / n_i)
//   B^H (spread) : g[l mod n] += f_j prod_i psi_i(x_ji - l_i / n_i)
// Reference: kernels.py:122-197 (gather_{1,2,3}d), :209-401 (spread_*).
//
// Both work on tile subproblems produced by the device sort (kernels.cu):
// one CTA per (tile, <= maxsub nodes).  The tile's (T + 2m + 1)^d halo lives
// in shared memory.  With T even the halo row length is odd, which keeps the
// lane-strided 128-bit row accesses bank-conflict free.
//
// Data movement: the interp halo arrives by TMA bulk copies (one
// cp.async.bulk per contiguous halo row, completion on an mbarrier); node
// batches (coordinates, samples, PRE_PSI factors) arrive by cp.async into a
// double buffer while the previous batch is being processed.
//
// Kernels are templated on the cutoff MM (1..8; 0 = runtime m) so the 2m-wide
// stencil loops unroll.  Nodes whose stencil is 2m+1 wide in some dimension
// (n x an exact integer, or fp rounding at the edges -- see common.cuh
// ``stencil``) take a generic path with runtime widths.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace nfftk {

__device__ __forceinline__ int wrapi(int v, int n) {
  v %= n;
  return v < 0 ? v + n : v;
}

__device__ __forceinline__ size_t a16(size_t v) { return (v + 15) & ~(size_t)15; }

template <int D>
__device__ __forceinline__ void tile_of(const Geom& g, int tile, int* tc, int* org) {
  int t = tile;
#pragma unroll
  for (int i = D - 1; i >= 0; --i) {
    tc[i] = t % g.ntile[i];
    t /= g.ntile[i];
  }
#pragma unroll
  for (int i = 0; i < D; ++i) org[i] = tc[i] * g.T[i] - g.m;
}

// wrapped grid slot of every halo coordinate, per dimension
template <int D>
__device__ __forceinline__ void build_slots(const Geom& g, const int* org, int* slots) {
  int off = 0;
#pragma unroll
  for (int dim = 0; dim < D; ++dim) {
    for (int a = threadIdx.x; a < g.H[dim]; a += blockDim.x) slots[off + a] = wrapi(org[dim] + a, g.n[dim]);
    off += g.H[dim];
  }
}

// ------------------------------------------------------- async copy PTX
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <typename C>
__device__ __forceinline__ void cp_async_cell(C* sdst, const C* gsrc) {
  if constexpr (sizeof(C) == 16) cp_async16(sdst, gsrc);
  else cp_async8(sdst, gsrc);
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared (size multiple of 16, both 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Halo staging.  complex128: one bulk copy per contiguous piece of a halo
// row (rows along the last dim; a row splits where it wraps).  complex64
// rows are not 16-byte multiples: per-cell cp.async.
template <typename C, int D>
__device__ __forceinline__ void issue_halo(const Geom& g, const C* __restrict__ grid, const int* slots,
                                           C* halo, unsigned long long* bar) {
  const int H0 = g.H[0];
  const int HL = g.H[D - 1];
  const int nl = g.n[D - 1];
  const int rows = D == 1 ? 1 : (D == 2 ? H0 : H0 * g.H[1]);
  const int* sl = slots + (D == 1 ? 0 : (D == 2 ? H0 : H0 + g.H[1]));
  if constexpr (sizeof(C) == 16) {
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      int64_t rbase = 0;
      if constexpr (D == 2) {
        rbase = (int64_t)slots[r] * g.n[1];
      } else if constexpr (D == 3) {
        int a = r / g.H[1], b = r - a * g.H[1];
        rbase = ((int64_t)slots[a] * g.n[1] + slots[H0 + b]) * g.n[2];
      }
      C* dst = halo + (size_t)r * HL;
      int c = 0;
      while (c < HL) {
        int s = sl[c];
        int len = min(HL - c, nl - s);
        bulk_g2s(dst + c, grid + rbase + s, (unsigned)(len * sizeof(C)), bar);
        c += len;
      }
    }
  } else {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (int r = warp; r < rows; r += nwarps) {
      int64_t rbase = 0;
      if constexpr (D == 2) {
        rbase = (int64_t)slots[r] * g.n[1];
      } else if constexpr (D == 3) {
        int a = r / g.H[1], b = r - a * g.H[1];
        rbase = ((int64_t)slots[a] * g.n[1] + slots[H0 + b]) * g.n[2];
      }
      for (int c = lane; c < HL; c += 32) cp_async_cell(halo + (size_t)r * HL + c, grid + rbase + sl[c]);
    }
  }
}

// Node batch buffers: coordinates, (interp) output index / (spread) sorted
// samples, window factors (copied from the PRE_PSI table, or computed) and
// per-node stencil data hw = {h_0..h_{D-1}, W_0..W_{D-1}, h_0 mod UA}.
template <typename C, int D>
struct Batch {
  double* x;   // [D][NB]
  double* w;   // [NB][D*K]
  int* hw;     // [NB][2D+1]
  int* pb;     // [NB] interp: output index
  C* fv;       // [NB] spread: sorted samples
};

__host__ __device__ inline size_t batch_bytes_of(int d, int nb, int K, int elem) {
  auto al = [](size_t v) { return (v + 15) & ~(size_t)15; };
  return al(sizeof(double) * d * nb) + al(sizeof(double) * nb * d * K) +
         al(sizeof(int) * nb * (2 * d + 1)) + al(sizeof(int) * nb) + al((size_t)elem * nb);
}

template <typename C, int D>
__device__ __forceinline__ Batch<C, D> batch_at(unsigned char* p, int nb, int K) {
  Batch<C, D> b;
  b.x = reinterpret_cast<double*>(p);
  p += a16(sizeof(double) * D * nb);
  b.w = reinterpret_cast<double*>(p);
  p += a16(sizeof(double) * nb * D * K);
  b.hw = reinterpret_cast<int*>(p);
  p += a16(sizeof(int) * nb * (2 * D + 1));
  b.pb = reinterpret_cast<int*>(p);
  p += a16(sizeof(int) * nb);
  b.fv = reinterpret_cast<C*>(p);
  return b;
}

// Issue the asynchronous copies of batch [base, base+nb).
template <typename C, int D>
__device__ __forceinline__ void issue_batch(const Geom& g, const double* __restrict__ xs,
                                            const int* __restrict__ perm, const C* __restrict__ fs,
                                            int base, int nb, int NB, const Batch<C, D>& b) {
  const int K = 2 * g.m + 1, per = D * K;
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
// in [0, T + m + 1], and (DIRECT / LUT) the window factors, from the staged
// coordinates (kernels.py:42-53 for a whole batch).  hw[2D] = h_0 mod ua.
template <typename C, int D>
__device__ __forceinline__ void finish_batch(const Geom& g, const int* tc, int nb, int NB, int ua,
                                             const Batch<C, D>& b) {
  const int K = 2 * g.m + 1, per = D * K;
  for (int q = threadIdx.x; q < nb * D; q += blockDim.x) {
    int j = q / D, dim = q - j * D;
    Stencil st = stencil(b.x[dim * NB + j], g.nd[dim], g.md);
    int slot = (int)floor_mod(st.cell, g.n[dim]);
    int h = slot - tc[dim] * g.T[dim] + g.m - (int)(st.cell - st.lo);
    b.hw[j * (2 * D + 1) + dim] = h;
    b.hw[j * (2 * D + 1) + D + dim] = st.width;
    if (dim == 0) b.hw[j * (2 * D + 1) + 2 * D] = h % ua;
  }
  if (g.mode != MODE_TENSOR) {
    for (int q = threadIdx.x; q < nb * per; q += blockDim.x) {
      int j = q / per, r = q - j * per, dim = r / K, t = r - dim * K;
      double x = b.x[dim * NB + j];
      Stencil st = stencil(x, g.nd[dim], g.md);
      b.w[q] = t < st.width ? dim_factor(g, dim, x, st.lo + t) * g.wscale[dim] : 0.0;
    }
  }
}

template <int D>
__device__ __forceinline__ bool is_fast(const int* q, int m) {
  bool f = true;
#pragma unroll
  for (int i = 0; i < D; ++i) f = f && q[D + i] == 2 * m;
  return f;
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
// One CTA per subproblem.  The halo arrives by TMA bulk copies while the first
// node batch arrives by cp.async; the next batch is fetched while the current
// one is processed.  A team of TEAM lanes reduces one node: lanes split the
// leading stencil dims and run along the contiguous last dim with the factors
// in registers; a team shuffle reduction forms f_j.
constexpr int INTERP_NB = 32;

template <typename R, int D, int MM>
__global__ void __launch_bounds__(512)
k_interp(const cplx_t<R>* __restrict__ grid, cplx_t<R>* __restrict__ fout,
         const double* __restrict__ xs, const int* __restrict__ perm,
         const int4* __restrict__ subs, Geom g) {
  using C = cplx_t<R>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int m = MM ? MM : g.m;
  const int K = 2 * m + 1;
  const int H0 = g.H[0], H1 = D > 1 ? g.H[1] : 1, H2 = D > 2 ? g.H[2] : 1;
  const int hsz = H0 * H1 * H2;
  const int nslots = H0 + (D > 1 ? H1 : 0) + (D > 2 ? H2 : 0);
  size_t off = 0;
  C* halo = reinterpret_cast<C*>(smem);
  off += a16((size_t)hsz * sizeof(C));
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + off);
  off += 16;
  int* slots = reinterpret_cast<int*>(smem + off);
  off += a16(nslots * sizeof(int));
  const size_t bb = batch_bytes_of(D, INTERP_NB, K, sizeof(C));
  Batch<C, D> buf[2] = {batch_at<C, D>(smem + off, INTERP_NB, K),
                        batch_at<C, D>(smem + off + bb, INTERP_NB, K)};
  constexpr int TEAM = InterpTeam<D, MM>::value;
  constexpr int NPW = 32 / TEAM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int tl = lane % TEAM, sub = lane / TEAM;
  const int4 sp = subs[blockIdx.x];
  int tc[D], org[D];
  tile_of<D>(g, sp.x, tc, org);
  build_slots<D>(g, org, slots);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    if (sizeof(C) == 16) mbar_expect_tx(bar, (unsigned)(hsz * sizeof(C)));
  }
  __syncthreads();
  issue_halo<C, D>(g, grid, slots, halo, bar);
  const int end = sp.y + sp.z;
  issue_batch<C, D>(g, xs, perm, nullptr, sp.y, min(INTERP_NB, sp.z), INTERP_NB, buf[0]);
  cp_async_commit();
  int k = 0;
  for (int base = sp.y; base < end; base += INTERP_NB, ++k) {
    const int nb = min(INTERP_NB, end - base);
    const Batch<C, D>& cur = buf[k & 1];
    cp_async_wait_all();
    __syncthreads();
    finish_batch<C, D>(g, tc, nb, INTERP_NB, 1, cur);
    __syncthreads();
    if (base + INTERP_NB < end) {
      issue_batch<C, D>(g, xs, perm, nullptr, base + INTERP_NB, min(INTERP_NB, end - base - INTERP_NB),
                        INTERP_NB, buf[(k + 1) & 1]);
      cp_async_commit();
    }
    if (k == 0 && sizeof(C) == 16) mbar_wait(bar, 0);
    for (int j0 = warp * NPW; j0 < nb; j0 += nwarps * NPW) {
      const int jb = j0 + sub;
      const bool active = jb < nb;
      const int* q = cur.hw + (active ? jb : j0) * (2 * D + 1);
      const double* w = cur.w + (active ? jb : j0) * D * K;
      R are = 0, aim = 0;
      if (active) {
        if (MM > 0 && is_fast<D>(q, m)) {
          constexpr int WF = 2 * (MM > 0 ? MM : 1);
          if constexpr (D == 1) {
            for (int t0 = tl; t0 < WF; t0 += TEAM) {
              C v = halo[q[0] + t0];
              R ww = (R)w[t0];
              are = fma(ww, v.x, are);
              aim = fma(ww, v.y, aim);
            }
          } else if constexpr (D == 2) {
            constexpr int SEG = WF / 2;
            for (int p = tl; p < 2 * WF; p += TEAM) {
              int t0 = p >> 1, seg = p & 1;
              const C* row = halo + (q[0] + t0) * H1 + q[1] + seg * SEG;
              const double* w1 = w + K + seg * SEG;
              R sre = 0, sim = 0;
#pragma unroll
              for (int t = 0; t < SEG; ++t) {
                C v = row[t];
                R ww = (R)w1[t];
                sre = fma(ww, v.x, sre);
                sim = fma(ww, v.y, sim);
              }
              R w0 = (R)w[t0];
              are = fma(w0, sre, are);
              aim = fma(w0, sim, aim);
            }
          } else {
            R w2r[WF];
#pragma unroll
            for (int t = 0; t < WF; ++t) w2r[t] = (R)w[2 * K + t];
            const C* corner = halo + (q[0] * H1 + q[1]) * H2 + q[2];
#pragma unroll 2
            for (int p = tl; p < WF * WF; p += TEAM) {
              int t0 = p / WF, t1 = p - t0 * WF;
              const C* row = corner + (t0 * H1 + t1) * H2;
              R sre = 0, sim = 0;
#pragma unroll
              for (int t = 0; t < WF; ++t) {
                C v = row[t];
                sre = fma(w2r[t], v.x, sre);
                sim = fma(w2r[t], v.y, sim);
              }
              R w01 = (R)(w[t0] * w[K + t1]);
              are = fma(w01, sre, are);
              aim = fma(w01, sim, aim);
            }
          }
        } else {
          // generic widths (2m or 2m+1 per dim), runtime loops
          if constexpr (D == 1) {
            for (int t0 = tl; t0 < q[1]; t0 += TEAM) {
              C v = halo[q[0] + t0];
              R ww = (R)w[t0];
              are = fma(ww, v.x, are);
              aim = fma(ww, v.y, aim);
            }
          } else {
            const int WL = q[2 * D - 1];
            const int P = D == 2 ? q[D] : q[D] * q[D + 1];
            const int W1 = D == 3 ? q[D + 1] : 1;
            const double* wl = w + (D - 1) * K;
            for (int p = tl; p < P; p += TEAM) {
              int t0 = p / W1, t1 = p - t0 * W1;
              const C* row = D == 2 ? halo + (q[0] + t0) * H1 + q[1]
                                    : halo + ((q[0] + t0) * H1 + q[1] + t1) * H2 + q[D - 1];
              R sre = 0, sim = 0;
              for (int t = 0; t < WL; ++t) {
                C v = row[t];
                sre = fma((R)wl[t], v.x, sre);
                sim = fma((R)wl[t], v.y, sim);
              }
              R wr = (R)(D == 2 ? w[t0] : w[t0] * w[K + t1]);
              are = fma(wr, sre, are);
              aim = fma(wr, sim, aim);
            }
          }
        }
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
        fout[cur.pb[jb]] = v;
      }
    }
  }
  if (sp.z <= 0 && sizeof(C) == 16) mbar_wait(bar, 0);
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
// Node batches (coordinates, sorted samples, factors) arrive by cp.async,
// double-buffered.  The finished halo is added to the HBM grid with fp64
// (fp32) RED atomics, skipping untouched cells.
constexpr int SPREAD_NB = 32;

template <typename R, int D, int MM>
__global__ void __launch_bounds__(512)
k_spread(cplx_t<R>* __restrict__ grid, const cplx_t<R>* __restrict__ fsorted,
         const double* __restrict__ xs, const int4* __restrict__ subs, Geom g) {
  using C = cplx_t<R>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int m = MM ? MM : g.m;
  const int K = 2 * m + 1;
  const int H0 = g.H[0], H1 = D > 1 ? g.H[1] : 1, H2 = D > 2 ? g.H[2] : 1;
  const int hsz = H0 * H1 * H2;
  const int nslots = H0 + (D > 1 ? H1 : 0) + (D > 2 ? H2 : 0);
  size_t off = 0;
  C* halo = reinterpret_cast<C*>(smem);
  off += a16((size_t)hsz * sizeof(C));
  int* slots = reinterpret_cast<int*>(smem + off);
  off += a16(nslots * sizeof(int));
  const size_t bb = batch_bytes_of(D, SPREAD_NB, K, sizeof(C));
  Batch<C, D> buf[2] = {batch_at<C, D>(smem + off, SPREAD_NB, K),
                        batch_at<C, D>(smem + off + bb, SPREAD_NB, K)};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int4 sp = subs[blockIdx.x];
  int tc[D], org[D];
  tile_of<D>(g, sp.x, tc, org);
  const int end = sp.y + sp.z;
  issue_batch<C, D>(g, xs, nullptr, fsorted, sp.y, min(SPREAD_NB, sp.z), SPREAD_NB, buf[0]);
  cp_async_commit();
  build_slots<D>(g, org, slots);
  for (int idx = threadIdx.x; idx < hsz; idx += blockDim.x) {
    C z;
    z.x = 0;
    z.y = 0;
    halo[idx] = z;
  }
  const int UA = D == 3 ? nwarps : (D == 2 ? (int)(blockDim.x >> 4) : (int)blockDim.x);
  int k = 0;
  for (int base = sp.y; base < end; base += SPREAD_NB, ++k) {
    const int nb = min(SPREAD_NB, end - base);
    const Batch<C, D>& cur = buf[k & 1];
    cp_async_wait_all();
    __syncthreads();  // batch k landed; previous batch applied; zeroing done
    finish_batch<C, D>(g, tc, nb, SPREAD_NB, UA, cur);
    __syncthreads();
    if (base + SPREAD_NB < end) {
      issue_batch<C, D>(g, xs, nullptr, fsorted, base + SPREAD_NB,
                        min(SPREAD_NB, end - base - SPREAD_NB), SPREAD_NB, buf[(k + 1) & 1]);
      cp_async_commit();
    }
    if constexpr (D == 3) {
      for (int jb = 0; jb < nb; ++jb) {
        const int* q = cur.hw + jb * (2 * D + 1);
        const int h0 = q[0], h1 = q[1], h2 = q[2], W0 = q[3], W1 = q[4], W2 = q[5];
        const double* w = cur.w + jb * D * K;
        const C f = cur.fv[jb];
        int d0 = warp - q[6];
        if (d0 < 0) d0 += UA;
        for (int a = h0 + d0; a < h0 + W0; a += UA) {
          R w0 = (R)w[a - h0];
          R cre = f.x * w0, cim = f.y * w0;
          C* plane = halo + (a * H1 + h1) * H2 + h2;
          if (MM > 0 && W1 == 2 * m && W2 == 2 * m) {
            constexpr int WF = 2 * (MM > 0 ? MM : 1);
#pragma unroll
            for (int p = lane; p < WF * WF; p += 32) {
              int t1 = p / WF, t2 = p - t1 * WF;
              R ww = (R)(w[K + t1] * w[2 * K + t2]);
              C* cell = plane + t1 * H2 + t2;
              C v = *cell;
              v.x = fma(cre, ww, v.x);
              v.y = fma(cim, ww, v.y);
              *cell = v;
            }
          } else {
            for (int p = lane; p < W1 * W2; p += 32) {
              int t1 = p / W2, t2 = p - t1 * W2;
              R ww = (R)(w[K + t1] * w[2 * K + t2]);
              C* cell = plane + t1 * H2 + t2;
              C v = *cell;
              v.x = fma(cre, ww, v.x);
              v.y = fma(cim, ww, v.y);
              *cell = v;
            }
          }
        }
        __syncwarp();
      }
    } else if constexpr (D == 2) {
      const int unit = threadIdx.x >> 4, U = UA, l16 = lane & 15;
      for (int jb = 0; jb < nb; ++jb) {
        const int* q = cur.hw + jb * (2 * D + 1);
        const int h0 = q[0], h1 = q[1], W0 = q[2], W1 = q[3];
        const double* w = cur.w + jb * D * K;
        const C f = cur.fv[jb];
        int d0 = unit - q[4];
        if (d0 < 0) d0 += U;
        for (int a = h0 + d0; a < h0 + W0; a += U) {
          R w0 = (R)w[a - h0];
          R cre = f.x * w0, cim = f.y * w0;
          C* row = halo + a * H1 + h1;
          for (int t1 = l16; t1 < W1; t1 += 16) {
            R ww = (R)w[K + t1];
            C v = row[t1];
            v.x = fma(cre, ww, v.x);
            v.y = fma(cim, ww, v.y);
            row[t1] = v;
          }
        }
        __syncwarp();
      }
    } else {
      const int unit = threadIdx.x, U = UA;
      for (int jb = 0; jb < nb; ++jb) {
        const int* q = cur.hw + jb * (2 * D + 1);
        const int h0 = q[0], W0 = q[1];
        const double* w = cur.w + jb * D * K;
        const C f = cur.fv[jb];
        int d0 = unit - q[2];
        if (d0 < 0) d0 += U;
        for (int a = h0 + d0; a < h0 + W0; a += U) {
          R w0 = (R)w[a - h0];
          C v = halo[a];
          v.x = fma(f.x, w0, v.x);
          v.y = fma(f.y, w0, v.y);
          halo[a] = v;
        }
      }
    }
  }
  __syncthreads();
  // ---- flush: rows of the halo, RED atomics into the wrapped grid slots
  if constexpr (D == 1) {
    for (int c = threadIdx.x; c < H0; c += blockDim.x) {
      C v = halo[c];
      if (v.x != (R)0 || v.y != (R)0) {
        atomicAdd(&grid[slots[c]].x, v.x);
        atomicAdd(&grid[slots[c]].y, v.y);
      }
    }
  } else {
    const int rows = D == 2 ? H0 : H0 * H1;
    const int HL = D == 2 ? H1 : H2;
    const int* sl = slots + H0 + (D == 3 ? H1 : 0);
    for (int r = warp; r < rows; r += nwarps) {
      int64_t rbase;
      if constexpr (D == 2) {
        rbase = (int64_t)slots[r] * g.n[1];
      } else {
        int a = r / H1, b = r - a * H1;
        rbase = ((int64_t)slots[a] * g.n[1] + slots[H0 + b]) * g.n[2];
      }
      for (int c = lane; c < HL; c += 32) {
        C v = halo[r * HL + c];
        if (v.x != (R)0 || v.y != (R)0) {
          C* dst = grid + rbase + sl[c];
          atomicAdd(&dst->x, v.x);
          atomicAdd(&dst->y, v.y);
        }
      }
    }
  }
}

// ================================================================ launchers
static size_t halo_cells(const Geom& g) {
  size_t h = 1;
  for (int i = 0; i < g.d; ++i) h *= g.H[i];
  return h;
}

static size_t slot_bytes(const Geom& g) {
  int s = 0;
  for (int i = 0; i < g.d; ++i) s += g.H[i];
  return (s * sizeof(int) + 15) & ~(size_t)15;
}

size_t interp_smem(const Geom& g, int elem_bytes, int threads) {
  (void)threads;
  size_t off = (halo_cells(g) * elem_bytes + 15) & ~(size_t)15;
  off += 16 + slot_bytes(g);
  off += 2 * batch_bytes_of(g.d, INTERP_NB, 2 * g.m + 1, elem_bytes);
  return off;
}

size_t spread_smem(const Geom& g, int elem_bytes) {
  size_t off = (halo_cells(g) * elem_bytes + 15) & ~(size_t)15;
  off += slot_bytes(g);
  off += 2 * batch_bytes_of(g.d, SPREAD_NB, 2 * g.m + 1, elem_bytes);
  return off;
}

int spread_threads(const Geom& g) {
  // d=3: one warp per owned a-row class (2m warps); d=2: 2m half-warp units;
  // d=1: 64 threads
  if (g.d == 3) return 32 * std::max(2, std::min(16, 2 * g.m));
  if (g.d == 2) return 16 * std::max(4, std::min(32, 2 * g.m));
  return 64;
}

template <typename R, int D, int MM>
static void interp_go(const void* grid, void* f, void*, const double* xs, const int* perm,
                      const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  const int threads = g.nt_interp;
  size_t smem = interp_smem(g, sizeof(cplx_t<R>), threads);
  auto kern = k_interp<R, D, MM>;
  NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<nsubs, threads, smem, s>>>((const cplx_t<R>*)grid, (cplx_t<R>*)f, xs, perm, subs, g);
  count_launch();
}

template <typename R, int D, int MM>
static void spread_go(void* grid, const void* f, void* fs, const double* xs, const int* perm,
                      const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  const int threads = spread_threads(g);
  size_t smem = spread_smem(g, sizeof(cplx_t<R>));
  auto kern = k_spread<R, D, MM>;
  NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_permute_samples<cplx_t<R>><<<(unsigned)std::min<int64_t>((g.M + 255) / 256, 148 * 64), 256, 0, s>>>(
      (const cplx_t<R>*)f, perm, g.M, (cplx_t<R>*)fs);
  count_launch();
  kern<<<nsubs, threads, smem, s>>>((cplx_t<R>*)grid, (const cplx_t<R>*)fs, xs, subs, g);
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

void launch_interp(bool single, const void* grid, void* f, const double* xs, const int* perm,
                   const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  if (nsubs <= 0) return;
  if (single) NFFTK_DISPATCH_DM(interp_go, float, grid, f, nullptr, xs, perm, subs, nsubs, g, s);
  else NFFTK_DISPATCH_DM(interp_go, double, grid, f, nullptr, xs, perm, subs, nsubs, g, s);
}

void launch_spread(bool single, void* grid, const void* f, void* fs, const double* xs,
                   const int* perm, const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  if (nsubs <= 0) return;
  if (single) NFFTK_DISPATCH_DM(spread_go, float, grid, f, fs, xs, perm, subs, nsubs, g, s);
  else NFFTK_DISPATCH_DM(spread_go, double, grid, f, fs, xs, perm, subs, nsubs, g, s);
}

}  // namespace nfftk
