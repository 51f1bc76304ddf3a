// sm_100a kernels of the nfftk hot path:
//   precompute : range check, tile binning keys, CUB radix sort, sorted node
//                coordinates, tile CSR + subproblem list, PRE_PSI table
//   D  / D^H   : deconvolution + zero-pad into the n-grid (fused k -> k mod n
//                slot mapping) and its transpose (pack + deconvolve)
//   B          : interpolation (gather) from a shared-memory tile halo
//   B^H        : spreading (scatter) into a shared-memory tile halo, flushed
//                to HBM with fp64 RED atomics
// Reference loops these replace: kernels.py:56-416, transform.py:39-176.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace nfftk {

// kernels launched by this library (any thread, any handle: atomic)
static std::atomic<unsigned long long> g_launches{0};
unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void add_launches(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// cells per segment when a line of len cells is cut into nseg warp-sized pieces
__host__ __device__ inline int seg_width(int len, int nseg) {
  return nseg <= 1 ? len : ((len + nseg - 1) / nseg + 31) / 32 * 32;
}

static inline unsigned blocks_for(int64_t work, int threads, int64_t cap = 148LL * 64) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

// ------------------------------------------------------------ validation
// plan.py:217-224 strict [-1/2, 1/2) check.  NaN fails the check here
// (the reference lets NaN through; on a device it would index out of bounds).
__global__ void k_check_range(const double* __restrict__ x, int64_t count,
                              unsigned long long* __restrict__ first_bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = x[i];
    if (!(v >= -0.5 && v < 0.5)) atomicMin(first_bad, (unsigned long long)i);
  }
}

void launch_check_range(const double* x, int64_t count, unsigned long long* first_bad,
                        cudaStream_t s) {
  k_check_range<<<blocks_for(count, 256), 256, 0, s>>>(x, count, first_bad);
  count_launch();
}

// ---------------------------------------------------------------- binning
// Sort key = tile-major cell index: tile (row-major over the tile grid) times
// T^d plus the cell's offset inside the tile, LAST dim most significant --
// nodes of a tile come grouped by their last-dim stencil offset, which the
// register-resident spread dispatches on once per run instead of per node.
// Cells are the slots floor(n x) mod n (kernels.py:47 wrapping, plan.py:229
// cell definition).
__global__ void k_bin_keys(const double* __restrict__ x, int64_t M, Geom g,
                           uint32_t* __restrict__ keys, int* __restrict__ vals,
                           int* __restrict__ tile_count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t tile = 0, local = 0, lc[MAX_D];
    for (int dim = 0; dim < g.d; ++dim) {
      double y = __dmul_rn(x[i * g.d + dim], g.nd[dim]);
      int64_t s = floor_mod((int64_t)floor(y), g.n[dim]);
      int tcoord = (int)(s / g.T[dim]);
      tile = tile * g.ntile[dim] + tcoord;
      lc[dim] = (uint32_t)(s - (int64_t)tcoord * g.T[dim]);
    }
    if (g.res) {
      // residue spread (residue.cu): ascending dim-0 cell (a lane changes rows
      // once per tile), runs of equal (dim-0, last-dim) cell inside it (one
      // unrolled FMA body per run), dim 1 least significant
      local = (lc[0] * 8 + lc[2]) * 8 + lc[1];
    } else {
      for (int dim = g.d - 1; dim >= 0; --dim) local = local * g.T[dim] + lc[dim];
    }
    uint32_t tvol = 1;
    for (int dim = 0; dim < g.d; ++dim) tvol *= g.T[dim];
    keys[i] = tile * tvol + local;
    vals[i] = (int)i;
    atomicAdd(&tile_count[tile], 1);
  }
}

__global__ void k_gather_sorted_x(const double* __restrict__ x, const int* __restrict__ perm,
                                  int64_t M, int d, double* __restrict__ xs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = perm[i];
    for (int dim = 0; dim < d; ++dim) xs[dim * M + i] = x[j * d + dim];
  }
}

__global__ void k_count_subs(const int* __restrict__ tile_count, int ntiles, int maxsub,
                             int* __restrict__ nsub) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ntiles) nsub[t] = (tile_count[t] + maxsub - 1) / maxsub;
}

__global__ void k_fill_subs(const int* __restrict__ tile_count, const int* __restrict__ tile_start,
                            const int* __restrict__ sub_start, int ntiles, int maxsub,
                            int4* __restrict__ subs) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  int c = tile_count[t], s0 = tile_start[t], o = sub_start[t];
  for (int k = 0; k * maxsub < c; ++k) {
    int cnt = c - k * maxsub;
    subs[o + k] = make_int4(t, s0 + k * maxsub, cnt < maxsub ? cnt : maxsub, 0);
  }
}

// Window evaluations per transform in DIRECT mode = sum of stencil widths
// (transform.py:116-117 counters).
__global__ void k_sum_widths(const double* __restrict__ xs, int64_t M, Geom g,
                             unsigned long long* __restrict__ total) {
  unsigned long long acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int dim = 0; dim < g.d; ++dim) acc += stencil(xs[dim * M + i], g.nd[dim], g.md).width;
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(total, acc);
}

// PRE_PSI table (kernels.py:56-72), sorted node order, zero-filled past width.
template <typename T>
__global__ void k_build_psi(const double* __restrict__ xs, int64_t M, Geom g,
                            T* __restrict__ psi) {
  const int K = 2 * g.m + 1, pr = g.pr;
  const int64_t total = M * pr;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = q / pr;
    int r = (int)(q - i * pr);
    int dim = 0, t = r;
    if (g.psi_pad == 1) {
      // halo-indexed leading dims, then the last dim's 2m+1 factors
      while (dim + 1 < g.d && t >= g.H[dim]) t -= g.H[dim++];
      if (dim + 1 == g.d && t >= K) dim = g.d;  // row padding
    } else if (g.psi_pad == 2) {
      // sten3 blocks of K + 1: last dim, dim 0, dim 1 (common.cuh)
      const int blk = r / (K + 1);
      t = r - blk * (K + 1);
      dim = blk == 0 ? g.d - 1 : (blk == 1 ? 0 : (blk == 2 ? 1 : g.d));
      if (t >= K) dim = g.d;  // the block's zero / row padding
    } else {
      dim = r / K;
      t = r - dim * K;
    }
    if (dim >= g.d) {
      psi[q] = 0.0;
      continue;
    }
    double x = xs[dim * M + i];
    Stencil st = stencil(x, g.nd[dim], g.md);
    if (g.psi_pad == 1 && dim + 1 < g.d) {
      // halo cell t -> stencil offset t - h (h as in k_build_recs)
      int64_t slot = floor_mod(st.cell, g.n[dim]);
      int tcoord = (int)(slot / g.T[dim]);
      int h = (int)(slot - (int64_t)tcoord * g.T[dim]) + g.m - (int)(st.cell - st.lo);
      t -= h;
      if (t < 0) {
        psi[q] = 0.0;
        continue;
      }
    }
    // factors are evaluated in fp64 (window.py:56-72) and rounded once to
    // the table type
    psi[q] = (T)(t < st.width ? dim_factor(g, dim, x, st.lo + t) * g.wscale[dim] : 0.0);
  }
}

// The same table, PSI_NODES rows per CTA: each (node, dim) stencil is formed
// once and its 2m+1 factors evaluated by consecutive threads into a zeroed
// shared-memory tile, which then leaves as one contiguous, coalesced block
// (the rows of consecutive sorted nodes are adjacent).  The per-entry kernel
// above re-derived the stencil for every table entry, zeros included.
constexpr int PSI_NODES = 64;
constexpr int PSI_STENCIL_BYTES = PSI_NODES * MAX_D * (8 + 4 + 4);
template <typename T>
__global__ void __launch_bounds__(256) k_build_psi_tile(const double* __restrict__ xs, int64_t M, Geom g,
                                                        T* __restrict__ psi) {
  extern __shared__ __align__(16) unsigned char psm[];
  // per (node, dim) stencil, formed once: lo, row position of offset 0, width
  int64_t* slo = reinterpret_cast<int64_t*>(psm);
  int* spos = reinterpret_cast<int*>(slo + PSI_NODES * MAX_D);
  int* swid = spos + PSI_NODES * MAX_D;
  T* tile = reinterpret_cast<T*>(psm + PSI_STENCIL_BYTES);
  const int K = 2 * g.m + 1, pr = g.pr;
  const int64_t i0 = (int64_t)blockIdx.x * PSI_NODES;
  const int nn = (int)min((int64_t)PSI_NODES, M - i0);
  for (int e = threadIdx.x; e < nn * pr; e += blockDim.x) tile[e] = (T)0;
  for (int nd = threadIdx.x; nd < nn * g.d; nd += blockDim.x) {
    const int dim = nd % g.d, j = nd / g.d;
    const Stencil st = stencil(xs[dim * M + i0 + j], g.nd[dim], g.md);
    int pos = dim * K;
    if (g.psi_pad == 1) {
      // halo-indexed leading dims (stencil offset t at halo cell h + t), then
      // the last dim's 2m+1 factors -- k_build_psi's layout
      int off = 0;
      for (int e = 0; e < dim; ++e) off += g.H[e];
      pos = off;
      if (dim + 1 < g.d) {
        const int64_t slot = floor_mod(st.cell, g.n[dim]);
        const int tcoord = (int)(slot / g.T[dim]);
        pos += (int)(slot - (int64_t)tcoord * g.T[dim]) + g.m - (int)(st.cell - st.lo);
      }
    } else if (g.psi_pad == 2) {
      // sten3 blocks: last dim, dim 0, dim 1 (common.cuh)
      pos = dim == g.d - 1 ? STEN3_OW2 : (dim == 0 ? sten3_ow0(K) : sten3_ow1(K));
    }
    slo[nd] = st.lo;
    spos[nd] = pos;
    swid[nd] = st.width;
  }
  __syncthreads();
  const int items = nn * g.d * K;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int t = it % K;
    const int nd = it / K;
    if (t >= swid[nd]) continue;
    const int dim = nd % g.d, j = nd / g.d;
    const double x = xs[dim * M + i0 + j];
    tile[j * pr + spos[nd] + t] = (T)(dim_factor(g, dim, x, slo[nd] + t) * g.wscale[dim]);
  }
  __syncthreads();
  T* out = psi + i0 * pr;
  for (int e = threadIdx.x; e < nn * pr; e += blockDim.x) out[e] = tile[e];
}

void build_psi(const double* xs, int64_t M, const Geom& g, void* psi, cudaStream_t s) {
  const size_t smem =
      PSI_STENCIL_BYTES + (size_t)PSI_NODES * g.pr * (g.psi_f32 ? sizeof(float) : sizeof(double));
  const unsigned blocks = (unsigned)((M + PSI_NODES - 1) / PSI_NODES);
  if (getenv("NFFTK_PSI_PER_ENTRY") || smem > 48 * 1024 || blocks == 0) {
    if (g.psi_f32)
      k_build_psi<float><<<blocks_for(M * g.pr, 256), 256, 0, s>>>(xs, M, g, (float*)psi);
    else
      k_build_psi<double><<<blocks_for(M * g.pr, 256), 256, 0, s>>>(xs, M, g, (double*)psi);
  } else if (g.psi_f32) {
    k_build_psi_tile<float><<<blocks, 256, smem, s>>>(xs, M, g, (float*)psi);
  } else {
    k_build_psi_tile<double><<<blocks, 256, smem, s>>>(xs, M, g, (double*)psi);
  }
  count_launch();
}

// Per-node stencil records in sorted order: halo-relative stencil starts
// h[dim] = (cell slot - tile start) + m - (cell - lo) and widths, packed
// {h0, h1, h2, W0 | W1 << 8 | W2 << 16 | fast << 24}.  The tile is the one
// k_bin_keys assigned (same slot arithmetic), so the spread reads one 16-byte
// record per node instead of recomputing stencils from coordinates.
__global__ void k_build_recs(const double* __restrict__ xs, int64_t M, Geom g,
                             int4* __restrict__ rec, unsigned* __restrict__ rrec,
                             unsigned* __restrict__ nwide) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    int h[3] = {0, 0, 0};
    unsigned packed = 0;
    bool fast = true;
    for (int dim = 0; dim < g.d; ++dim) {
      Stencil st = stencil(xs[dim * M + i], g.nd[dim], g.md);
      int64_t slot = floor_mod(st.cell, g.n[dim]);
      int tcoord = (int)(slot / g.T[dim]);
      h[dim] = (int)(slot - (int64_t)tcoord * g.T[dim]) + g.m - (int)(st.cell - st.lo);
      packed |= (unsigned)st.width << (8 * dim);
      fast = fast && st.width == 2 * g.m;
    }
    packed |= (unsigned)fast << 24;
    rec[i] = make_int4(h[0], h[1], h[2], (int)packed);
    if (rrec) {
      // residue record (common.cuh RES_*): a regular node's halo start is its
      // cell inside the tile (h - 1 in the 15^3 halo)
      rrec[i] = fast ? ((unsigned)(h[0] - 1) | (unsigned)(h[1] - 1) << 3 | (unsigned)(h[2] - 1) << 6 | RES_REGULAR) : 0u;
      if (!fast) atomicAdd(nwide, 1u);
    }
  }
}

void build_recs(const double* xs, int64_t M, const Geom& g, int4* rec, unsigned* rrec, unsigned* nwide,
                cudaStream_t s) {
  k_build_recs<<<blocks_for(M, 256), 256, 0, s>>>(xs, M, g, rec, rrec, nwide);
  count_launch();
}

// PrecomputeTables.psi in the reference layout (plan.py:109-121, :258-266;
// kernels.py:56-72): out[j, i, t] = window(x_ji - (lo_ji + t) / n_i) for t <
// width, 0 beyond, natural node order, exact fp64 factors (no complex64
// normalisation, no LUT).  Built on demand for callers that inspect it.
__global__ void k_psi_reference(const double* __restrict__ x, int64_t M, Geom g, double* __restrict__ out) {
  const int K = 2 * g.m + 1;
  const int64_t total = M * g.d * K;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ji = q / K;
    const int t = (int)(q - ji * K);
    const int i = (int)(ji % g.d);
    const double xv = x[ji];
    const Stencil st = stencil(xv, g.nd[i], g.md);
    double v = 0.0;
    if (t < st.width) {
      const double off = __dsub_rn(xv, (double)(st.lo + t) / g.nd[i]);
      v = g.code == WINDOW_KB ? window_kb(off, g.nd[i], g.md, g.b[i]) : window_gauss(off, g.nd[i], g.b[i]);
    }
    out[q] = v;
  }
}

// PRE_FULL_PSI tables in the reference layout (kernels.py:85-119): per node
// the (2m+1)^d slots of products ((f0 f1) f2) over the stencil in
// lexicographic order and their flat wrapped grid cells; slots past the
// node's count stay zero (plan.py:270-279 zero-initialises both).
__global__ void k_psi_full_reference(const double* __restrict__ psi, const double* __restrict__ x, int64_t M,
                                     Geom g, double* __restrict__ vals, int64_t* __restrict__ idx,
                                     int64_t* __restrict__ counts) {
  const int K = 2 * g.m + 1;
  int64_t P = 1;
  for (int i = 0; i < g.d; ++i) P *= K;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo[MAX_D];
    int W[MAX_D] = {1, 1, 1};
    for (int i = 0; i < g.d; ++i) {
      const Stencil st = stencil(x[j * g.d + i], g.nd[i], g.md);
      lo[i] = st.lo;
      W[i] = st.width;
    }
    const double* f = psi + j * g.d * K;
    double* vo = vals + j * P;
    int64_t* io = idx + j * P;
    int64_t p = 0;
    for (int t0 = 0; t0 < W[0]; ++t0) {
      const int64_t r0 = floor_mod(lo[0] + t0, g.n[0]);
      if (g.d == 1) { vo[p] = f[t0]; io[p++] = r0; continue; }
      for (int t1 = 0; t1 < W[1]; ++t1) {
        const int64_t r1 = floor_mod(lo[1] + t1, g.n[1]);
        const double f01 = __dmul_rn(f[t0], f[K + t1]);
        if (g.d == 2) { vo[p] = f01; io[p++] = r0 * g.n[1] + r1; continue; }
        const int64_t r01 = (r0 * g.n[1] + r1) * g.n[2];
        for (int t2 = 0; t2 < W[2]; ++t2) {
          vo[p] = __dmul_rn(f01, f[2 * K + t2]);
          io[p++] = r01 + floor_mod(lo[2] + t2, g.n[2]);
        }
      }
    }
    for (; p < P; ++p) { vo[p] = 0.0; io[p] = 0; }
    int64_t c = 1;
    for (int i = 0; i < g.d; ++i) c *= W[i];
    counts[j] = c;
  }
}

void psi_reference(const double* x_dev, int64_t M, const Geom& g, double* psi, double* vals, int64_t* idx,
                   int64_t* counts, cudaStream_t s) {
  k_psi_reference<<<blocks_for(M * g.d * (2 * g.m + 1), 256), 256, 0, s>>>(x_dev, M, g, psi);
  count_launch();
  if (vals) {
    k_psi_full_reference<<<blocks_for(M, 128), 128, 0, s>>>(psi, x_dev, M, g, vals, idx, counts);
    count_launch();
  }
}

// Lexicographic cell order (plan.py:228-231): stable sort of (floor(n x)
// row-major key, index) reproduces np.lexsort exactly.
__global__ void k_lex_keys(const double* __restrict__ x, int64_t M, Geom g,
                           unsigned long long* __restrict__ keys, int* __restrict__ vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long k = 0;
    for (int dim = 0; dim < g.d; ++dim) {
      int64_t c = (int64_t)floor(__dmul_rn(x[i * g.d + dim], g.nd[dim])) + g.n[dim] / 2;
      k = k * (unsigned long long)(g.n[dim] + 1) + (unsigned long long)c;
    }
    keys[i] = k;
    vals[i] = (int)i;
  }
}

static int bits_for(unsigned long long v) {
  int b = 0;
  while (b < 64 && (1ULL << b) < v) ++b;
  return b < 1 ? 1 : b;
}

// weight class of a subproblem, 0 = heaviest (count near maxsub)
__global__ void k_sub_keys(const int4* __restrict__ subs, int total, int maxsub,
                           uint32_t* __restrict__ keys, int* __restrict__ vals) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  keys[i] = (uint32_t)(((int64_t)(maxsub - subs[i].z) * 8) / (maxsub + 1));
  vals[i] = i;
}

// d = 3: subproblems in blocks of 4 x 4 x ntile[2] tiles
// (dim-0 / dim-1 neighbours stay within ~256 subproblems, so the halo overlap
// of neighbouring tiles -- the spread's reductions, the interp's box loads --
// meets in L2 instead of HBM), in three weight classes around the mean count
// so that evenly filled tiles keep one order.
__global__ void k_sub_keys_res(const int4* __restrict__ subs, int total, int mean, Geom g,
                               uint32_t* __restrict__ keys, int* __restrict__ vals) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int4 sp = subs[i];
  int t = sp.x;
  const int k = t % g.ntile[2];
  t /= g.ntile[2];
  const int j = t % g.ntile[1], a = t / g.ntile[1];
  const uint32_t nb1 = (uint32_t)(g.ntile[1] + 3) / 4;
  const uint32_t blk = ((uint32_t)(a / 4) * nb1 + (uint32_t)(j / 4)) * 16u + (uint32_t)((a % 4) * 4 + (j % 4));
  const uint32_t cls = sp.z > 2 * mean ? 0u : (2 * sp.z >= mean ? 1u : 2u);
  const uint32_t nblk = (uint32_t)((g.ntile[0] + 3) / 4) * nb1 * 16u;
  keys[i] = (cls * nblk + blk) * (uint32_t)g.ntile[2] + (uint32_t)k;
  vals[i] = i;
}

__global__ void k_gather_subs(const int4* __restrict__ subs, const int* __restrict__ order, int total,
                              int4* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) out[i] = subs[order[i]];
}

// The sort's temporaries come from the device's default stream-ordered pool;
// with its default release threshold (0) every synchronisation hands the
// memory back and the next set_nodes maps it again (~60 us per
// cudaMallocAsync).  Keep what the pool holds (at most the largest set_nodes'
// temporaries: keys, values, CUB workspace).
static void keep_pool_memory() {
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done[dev] = true;
}

void bin_and_sort(const double* x_dev, int64_t M, const Geom& g, int maxsub, int ntiles,
                  int* perm, double* xs, int* tile_count, int* tile_start, int4** subs,
                  int* nsubs, cudaStream_t s) {
  keep_pool_memory();
  uint32_t *keys = nullptr, *keys2 = nullptr;
  int *vals = nullptr, *nsub = nullptr, *sub_start = nullptr;
  NFFTK_CUDA(cudaMallocAsync(&keys, sizeof(uint32_t) * M * 2, s));
  keys2 = keys + M;
  NFFTK_CUDA(cudaMallocAsync(&vals, sizeof(int) * M, s));
  NFFTK_CUDA(cudaMemsetAsync(tile_count, 0, sizeof(int) * (ntiles + 1), s));
  k_bin_keys<<<blocks_for(M, 256), 256, 0, s>>>(x_dev, M, g, keys, vals, tile_count);
  count_launch();
  unsigned long long keyspace = 1;
  for (int i = 0; i < g.d; ++i) keyspace *= (unsigned long long)g.ntile[i] * g.T[i];
  int end_bit = bits_for(keyspace);
  size_t tmp_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, vals, perm, (int)M, 0, end_bit, s);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, tile_count, tile_start, ntiles + 1, s);
  size_t need = tmp_bytes > scan_bytes ? tmp_bytes : scan_bytes;
  void* tmp = nullptr;
  NFFTK_CUDA(cudaMallocAsync(&tmp, need, s));
  NFFTK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, perm, (int)M, 0,
                                             end_bit, s));
  count_launch();
  k_gather_sorted_x<<<blocks_for(M, 256), 256, 0, s>>>(x_dev, perm, M, g.d, xs);
  count_launch();
  NFFTK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, tile_count, tile_start, ntiles + 1, s));
  count_launch();
  // subproblems: ceil(count / maxsub) per tile
  NFFTK_CUDA(cudaMallocAsync(&nsub, sizeof(int) * (ntiles + 1) * 2, s));
  sub_start = nsub + ntiles + 1;
  NFFTK_CUDA(cudaMemsetAsync(nsub, 0, sizeof(int) * (ntiles + 1), s));
  k_count_subs<<<(ntiles + 255) / 256, 256, 0, s>>>(tile_count, ntiles, maxsub, nsub);
  count_launch();
  NFFTK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, nsub, sub_start, ntiles + 1, s));
  count_launch();
  int total = 0;
  NFFTK_CUDA(cudaMemcpyAsync(&total, sub_start + ntiles, sizeof(int), cudaMemcpyDeviceToHost, s));
  NFFTK_CUDA(cudaStreamSynchronize(s));
  if (*subs) NFFTK_CUDA(cudaFree(*subs));
  *subs = nullptr;
  NFFTK_CUDA(cudaMalloc(subs, sizeof(int4) * (total > 0 ? total : 1)));
  k_fill_subs<<<(ntiles + 255) / 256, 256, 0, s>>>(tile_count, tile_start, sub_start, ntiles,
                                                   maxsub, *subs);
  count_launch();
  *nsubs = total;
  // heaviest subproblems first, in 8 weight classes (ties keep tile order):
  // with clustered nodes the last subproblems a persistent CTA draws are
  // then light, which shortens the tail; evenly filled tiles all land in one
  // class and keep their order
  if (total > 1 && !getenv("NFFTK_NO_LPT")) {
    uint32_t* sk = nullptr;
    int* sv = nullptr;
    int4* sorted = nullptr;
    NFFTK_CUDA(cudaMallocAsync(&sk, sizeof(uint32_t) * total * 2, s));
    NFFTK_CUDA(cudaMallocAsync(&sv, sizeof(int) * total * 2, s));
    NFFTK_CUDA(cudaMalloc(&sorted, sizeof(int4) * total));
    int key_bits = 3;
    if (g.d == 3 && !getenv("NFFTK_NO_BLOCK_ORDER")) {
      const int mean = (int)std::max<int64_t>(1, M / std::max(1, ntiles));
      k_sub_keys_res<<<(total + 255) / 256, 256, 0, s>>>(*subs, total, mean, g, sk, sv);
      key_bits = bits_for(3ull * ((g.ntile[0] + 3) / 4) * ((g.ntile[1] + 3) / 4) * 16ull * g.ntile[2]);
    } else {
      k_sub_keys<<<(total + 255) / 256, 256, 0, s>>>(*subs, total, maxsub, sk, sv);
    }
    count_launch();
    size_t lb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, lb, sk, sk + total, sv, sv + total, total, 0, key_bits, s);
    void* ltmp = nullptr;
    NFFTK_CUDA(cudaMallocAsync(&ltmp, lb, s));
    NFFTK_CUDA(cub::DeviceRadixSort::SortPairs(ltmp, lb, sk, sk + total, sv, sv + total, total, 0, key_bits, s));
    count_launch();
    k_gather_subs<<<(total + 255) / 256, 256, 0, s>>>(*subs, sv + total, total, sorted);
    count_launch();
    NFFTK_CUDA(cudaFreeAsync(ltmp, s));
    NFFTK_CUDA(cudaFreeAsync(sv, s));
    NFFTK_CUDA(cudaFreeAsync(sk, s));
    NFFTK_CUDA(cudaStreamSynchronize(s));
    NFFTK_CUDA(cudaFree(*subs));
    *subs = sorted;
  }
  NFFTK_CUDA(cudaFreeAsync(tmp, s));
  NFFTK_CUDA(cudaFreeAsync(nsub, s));
  NFFTK_CUDA(cudaFreeAsync(vals, s));
  NFFTK_CUDA(cudaFreeAsync(keys, s));
}

unsigned long long sum_widths(const double* xs, int64_t M, const Geom& g, cudaStream_t s) {
  unsigned long long* d_total = nullptr;
  unsigned long long total = 0;
  NFFTK_CUDA(cudaMallocAsync(&d_total, sizeof(unsigned long long), s));
  NFFTK_CUDA(cudaMemsetAsync(d_total, 0, sizeof(unsigned long long), s));
  k_sum_widths<<<blocks_for(M, 256), 256, 0, s>>>(xs, M, g, d_total);
  count_launch();
  NFFTK_CUDA(cudaMemcpyAsync(&total, d_total, sizeof(total), cudaMemcpyDeviceToHost, s));
  NFFTK_CUDA(cudaFreeAsync(d_total, s));
  NFFTK_CUDA(cudaStreamSynchronize(s));
  return total;
}


void lex_order(const double* x_dev, int64_t M, const Geom& g, int* order, cudaStream_t s) {
  unsigned long long *keys = nullptr;
  int* vals = nullptr;
  NFFTK_CUDA(cudaMallocAsync(&keys, sizeof(unsigned long long) * M * 2, s));
  NFFTK_CUDA(cudaMallocAsync(&vals, sizeof(int) * M, s));
  k_lex_keys<<<blocks_for(M, 256), 256, 0, s>>>(x_dev, M, g, keys, vals);
  count_launch();
  unsigned long long keyspace = 1;
  for (int i = 0; i < g.d; ++i) keyspace *= (unsigned long long)(g.n[i] + 1);
  int end_bit = bits_for(keyspace);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys + M, vals, order, (int)M, 0,
                                  end_bit, s);
  void* tmp = nullptr;
  NFFTK_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
  NFFTK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys + M, vals, order, (int)M,
                                             0, end_bit, s));
  count_launch();
  NFFTK_CUDA(cudaFreeAsync(tmp, s));
  NFFTK_CUDA(cudaFreeAsync(vals, s));
  NFFTK_CUDA(cudaFreeAsync(keys, s));
}

// ------------------------------------------------------------ D and D^H
// transform.py:57-63 + :96-97: g[k mod n] = f_hat_k / (|I_n| prod_i phi_hat_i)
// and zero elsewhere; transform.py:174-176 applies the same scaling to the
// packed g.  The reciprocal factors are tabulated at precompute; the
// product 1/|I_n| * prod 1/phi_hat differs from the reference's sequence of
// divisions only in the last bits (~4 ulp).  One warp per grid line (lanes
// along the contiguous last dim), eight lines per 256-thread block.
struct DeconvGeom {
  int d;
  int N[MAX_D];
  int n[MAX_D];
  const double* icol[MAX_D];  // 1 / (phi_hat * wscale) over k + N/2
  double inv_gs;              // 1 / |I_n|
};

template <typename R>
__global__ void __launch_bounds__(256) k_deconv_pad(const cplx_t<R>* __restrict__ fhat,
                                                    cplx_t<R>* __restrict__ grid, DeconvGeom q,
                                                    int64_t lines, int nseg) {
  using C = cplx_t<R>;
  const int dl = q.d - 1;
  const int nl = q.n[dl], Nl = q.N[dl], h = Nl / 2;
  const int lane = threadIdx.x & 31;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int segw = seg_width(nl, nseg);
  for (int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < lines * nseg;
       item += wstride) {
    const int64_t line = item / nseg;
    const int s0 = (int)(item - line * nseg) * segw, s1 = min(nl, s0 + segw);
    bool inside = true;
    int64_t fl = 0, rem = line;
    double fac = q.inv_gs;
    int lead[MAX_D];
    for (int i = dl - 1; i >= 0; --i) { lead[i] = (int)(rem % q.n[i]); rem /= q.n[i]; }
    for (int i = 0; i < dl; ++i) {
      int sl = lead[i], Ni = q.N[i];
      int k = sl < Ni / 2 ? sl + Ni / 2 : (sl >= q.n[i] - Ni / 2 ? sl - q.n[i] + Ni / 2 : -1);
      inside = inside && k >= 0;
      fl = fl * Ni + (k < 0 ? 0 : k);
      if (k >= 0) fac *= q.icol[i][k];
    }
    C* out = grid + line * nl;
    const C* in = fhat + fl * Nl;
    for (int sl = s0 + lane; sl < s1; sl += 32) {
      C v;
      v.x = 0;
      v.y = 0;
      int k = sl < h ? sl + h : (sl >= nl - h ? sl - nl + h : -1);
      if (inside && k >= 0) {
        C a = in[k];
        double f = fac * q.icol[dl][k];
        v.x = (R)((double)a.x * f);
        v.y = (R)((double)a.y * f);
      }
      out[sl] = v;
    }
  }
}

template <typename R>
__global__ void __launch_bounds__(256) k_pack_deconv(const cplx_t<R>* __restrict__ grid,
                                                     cplx_t<R>* __restrict__ fhat, DeconvGeom q,
                                                     int64_t lines, int nseg) {
  using C = cplx_t<R>;
  const int dl = q.d - 1;
  const int nl = q.n[dl], Nl = q.N[dl];
  const int lane = threadIdx.x & 31;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int segw = seg_width(Nl, nseg);
  for (int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < lines * nseg;
       item += wstride) {
    const int64_t line = item / nseg;
    const int s0 = (int)(item - line * nseg) * segw, s1 = min(Nl, s0 + segw);
    int64_t gl = 0, rem = line;
    double fac = q.inv_gs;
    int kidx[MAX_D];
    for (int i = dl - 1; i >= 0; --i) { kidx[i] = (int)(rem % q.N[i]); rem /= q.N[i]; }
    for (int i = 0; i < dl; ++i) {
      int k = kidx[i] - q.N[i] / 2;
      gl = gl * q.n[i] + (k < 0 ? k + q.n[i] : k);
      fac *= q.icol[i][kidx[i]];
    }
    const C* in = grid + gl * nl;
    C* out = fhat + line * Nl;
    for (int kl = s0 + lane; kl < s1; kl += 32) {
      int k = kl - Nl / 2;
      C a = in[k < 0 ? k + nl : k];
      double f = fac * q.icol[dl][kl];
      C v;
      v.x = (R)((double)a.x * f);
      v.y = (R)((double)a.y * f);
      out[kl] = v;
    }
  }
}

static unsigned line_blocks(int64_t lines) {
  int64_t b = (lines + 7) / 8;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148LL * 16));
}

// Segments per line for the warp-per-line kernels: few, long lines (d = 1:
// one line) are cut into 32-cell multiples so a small grid still spreads
// over the SMs (C1: one warp walked all 2048 cells of the only line).
static int line_segments(int64_t lines, int len) {
  const int64_t target = 148LL * 64;  // warps
  int64_t seg = std::max<int64_t>(1, target / std::max<int64_t>(1, lines));
  return (int)std::min<int64_t>(seg, (len + 31) / 32);
}

template <typename R>
void launch_deconv_pad(const void* fhat, void* grid, const DeconvGeom& q, cudaStream_t s) {
  int64_t lines = 1;
  for (int i = 0; i < q.d - 1; ++i) lines *= q.n[i];
  const int nseg = line_segments(lines, q.n[q.d - 1]);
  k_deconv_pad<R><<<line_blocks(lines * nseg), 256, 0, s>>>((const cplx_t<R>*)fhat, (cplx_t<R>*)grid, q,
                                                            lines, nseg);
  count_launch();
}

template <typename R>
void launch_pack_deconv(const void* grid, void* fhat, const DeconvGeom& q, cudaStream_t s) {
  int64_t lines = 1;
  for (int i = 0; i < q.d - 1; ++i) lines *= q.N[i];
  const int nseg = line_segments(lines, q.N[q.d - 1]);
  k_pack_deconv<R><<<line_blocks(lines * nseg), 256, 0, s>>>((const cplx_t<R>*)grid, (cplx_t<R>*)fhat, q,
                                                             lines, nseg);
  count_launch();
}

void launch_deconv(bool single, const void* fhat, void* grid, const DeconvGeomH& qh, cudaStream_t s) {
  DeconvGeom q;
  q.d = qh.d;
  for (int i = 0; i < MAX_D; ++i) { q.N[i] = qh.N[i]; q.n[i] = qh.n[i]; q.icol[i] = qh.icol[i]; }
  q.inv_gs = 1.0 / qh.grid_size;
  if (single) launch_deconv_pad<float>(fhat, grid, q, s);
  else launch_deconv_pad<double>(fhat, grid, q, s);
}

void launch_pack(bool single, const void* grid, void* fhat, const DeconvGeomH& qh, cudaStream_t s) {
  DeconvGeom q;
  q.d = qh.d;
  for (int i = 0; i < MAX_D; ++i) { q.N[i] = qh.N[i]; q.n[i] = qh.n[i]; q.icol[i] = qh.icol[i]; }
  q.inv_gs = 1.0 / qh.grid_size;
  if (single) launch_pack_deconv<float>(grid, fhat, q, s);
  else launch_pack_deconv<double>(grid, fhat, q, s);
}

}  // namespace nfftk

namespace nfftk {
// ------------------------------------------------- FMA peak microbenchmark
// Measures the FP64 / FP32 FMA roof that bounds the c128 / c64 gridding
// kernels (MEASURED_PEAKS.json only carries HBM and bf16 figures).
template <typename T>
__global__ void k_fma_peak(T* out, int iters) {
  T a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = (T)(threadIdx.x + k) * (T)1e-3;
  const T b = (T)0.999999, c = (T)1e-6;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  T s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == (T)-1) out[0] = s;  // never true; keeps the chains alive
}

double measure_fma_tflops(bool fp64) {
  int dev = 0, sms = 0;
  NFFTK_CUDA(cudaGetDevice(&dev));
  NFFTK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  void* out = nullptr;
  NFFTK_CUDA(cudaMalloc(&out, 16));
  const int threads = 256, blocks = sms * 8, iters = fp64 ? 8192 : 32768;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    if (fp64) k_fma_peak<double><<<blocks, threads>>>((double*)out, iters);
    else k_fma_peak<float><<<blocks, threads>>>((float*)out, iters);
    cudaEventRecord(b);
    NFFTK_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    double tf = flops / (ms * 1e-3) / 1e12;
    if (rep > 0 && tf > best) best = tf;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  return best;
}
}  // namespace nfftk

namespace nfftk {
// ----------------------------------------------- ghost-padded grid copies
// The padded grid holds cell slot s of the n-grid at padded index s + m and
// periodic images in the ghost layers, so every tile halo [t T - m, t T + T
// + m] is one contiguous box at padded origin t T.

// dense -> padded (after the forward FFT): every padded cell reads its image
__device__ __forceinline__ int wrap_slot(int p, int m, int n) {
  int s = p - m;  // the padded extent keeps p - m in [-n, 2n) (plan.cu)
  if (s < 0) s += n;
  if (s >= n) s -= n;
  return s;
}

template <typename C>
__global__ void __launch_bounds__(256) k_pad(const C* __restrict__ g0, C* __restrict__ gp, PadGeom q,
                                             int lines, int nseg) {
  const int dl = q.d - 1;
  const int nl = q.n[dl], npl = q.np[dl];
  const int lane = threadIdx.x & 31;
  const int wstride = (gridDim.x * blockDim.x) >> 5;
  const int segw = seg_width(npl, nseg);
  for (int item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < lines * nseg; item += wstride) {
    const int line = item / nseg;
    const int s0 = (item - line * nseg) * segw, s1 = min(npl, s0 + segw);
    int src = 0, rem = line;
    int lead[MAX_D];
    for (int i = dl - 1; i >= 0; --i) { lead[i] = rem % q.np[i]; rem /= q.np[i]; }
    for (int i = 0; i < dl; ++i) src = src * q.n[i] + wrap_slot(lead[i], q.m, q.n[i]);
    const C* in = g0 + (int64_t)src * nl;
    C* out = gp + (int64_t)line * npl;
    for (int p = s0 + lane; p < s1; p += 32) out[p] = in[wrap_slot(p, q.m, nl)];
  }
}

// padded -> dense (after the spread): each dense cell sums its images
template <typename C>
__global__ void __launch_bounds__(256) k_fold(const C* __restrict__ gp, C* __restrict__ g0, PadGeom q,
                                              int lines, int nseg) {
  const int dl = q.d - 1;
  const int nl = q.n[dl], npl = q.np[dl];
  const int lane = threadIdx.x & 31;
  const int wstride = (gridDim.x * blockDim.x) >> 5;
  const int segw = seg_width(nl, nseg);
  for (int item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < lines * nseg; item += wstride) {
    const int line = item / nseg;
    const int s0 = (item - line * nseg) * segw, s1 = min(nl, s0 + segw);
    int rem = line;
    int c[MAX_D];
    for (int i = dl - 1; i >= 0; --i) { c[i] = rem % q.n[i]; rem /= q.n[i]; }
    // padded lines holding images of this dense line (<= 3 per leading dim)
    int64_t plines[9];
    int np_lines = 1;
    plines[0] = 0;
    for (int i = 0; i < dl; ++i) {
      int cand[3], nc = 0;
      for (int k = -1; k <= 1; ++k) {
        int p = c[i] + q.m + k * q.n[i];
        if (p >= 0 && p < q.np[i]) cand[nc++] = p;
      }
      int64_t tmp[9];
      int nt = 0;
      for (int a2 = 0; a2 < np_lines; ++a2)
        for (int b2 = 0; b2 < nc && nt < 9; ++b2) tmp[nt++] = plines[a2] * q.np[i] + cand[b2];
      for (int a2 = 0; a2 < nt; ++a2) plines[a2] = tmp[a2];
      np_lines = nt;
    }
    C* out = g0 + (int64_t)line * nl;
    for (int s2 = s0 + lane; s2 < s1; s2 += 32) {
      double re = 0, im = 0;
      const int p0 = s2 + q.m;
      const bool lo_img = p0 - nl >= 0, hi_img = p0 + nl < npl;
      for (int a2 = 0; a2 < np_lines; ++a2) {
        const C* row = gp + plines[a2] * npl;
        C v = row[p0];
        re += (double)v.x;
        im += (double)v.y;
        if (lo_img) {
          v = row[p0 - nl];
          re += (double)v.x;
          im += (double)v.y;
        }
        if (hi_img) {
          v = row[p0 + nl];
          re += (double)v.x;
          im += (double)v.y;
        }
      }
      C v;
      v.x = (decltype(v.x))re;
      v.y = (decltype(v.y))im;
      out[s2] = v;
    }
  }
}

void launch_pad(bool single, const void* g0, void* gp, const PadGeom& q, cudaStream_t s) {
  int64_t lines = 1;
  for (int i = 0; i < q.d - 1; ++i) lines *= q.np[i];
  const int nseg = line_segments(lines, q.np[q.d - 1]);
  const unsigned nb = line_blocks(lines * nseg);
  if (single) k_pad<float2><<<nb, 256, 0, s>>>((const float2*)g0, (float2*)gp, q, (int)lines, nseg);
  else k_pad<double2><<<nb, 256, 0, s>>>((const double2*)g0, (double2*)gp, q, (int)lines, nseg);
  count_launch();
}

void launch_fold(bool single, const void* gp, void* g0, const PadGeom& q, cudaStream_t s) {
  int64_t lines = 1;
  for (int i = 0; i < q.d - 1; ++i) lines *= q.n[i];
  const int nseg = line_segments(lines, q.n[q.d - 1]);
  const unsigned nb = line_blocks(lines * nseg);
  if (single) k_fold<float2><<<nb, 256, 0, s>>>((const float2*)gp, (float2*)g0, q, (int)lines, nseg);
  else k_fold<double2><<<nb, 256, 0, s>>>((const double2*)gp, (double2*)g0, q, (int)lines, nseg);
  count_launch();
}
}  // namespace nfftk
