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

#include "common.cuh"
#include "kernels.h"

namespace nfftk {

static unsigned long long g_launches = 0;  // kernels launched by this library
unsigned long long launch_count() { return g_launches; }
static inline void count_launch() { ++g_launches; }

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
// T^d plus the cell's row-major offset inside the tile.  Cells are the slots
// floor(n x) mod n (kernels.py:47 wrapping, plan.py:229 cell definition).
__global__ void k_bin_keys(const double* __restrict__ x, int64_t M, Geom g,
                           uint32_t* __restrict__ keys, int* __restrict__ vals,
                           int* __restrict__ tile_count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t tile = 0, local = 0;
    for (int dim = 0; dim < g.d; ++dim) {
      double y = __dmul_rn(x[i * g.d + dim], g.nd[dim]);
      int64_t s = floor_mod((int64_t)floor(y), g.n[dim]);
      int tcoord = (int)(s / g.T[dim]);
      tile = tile * g.ntile[dim] + tcoord;
      local = local * g.T[dim] + (uint32_t)(s - (int64_t)tcoord * g.T[dim]);
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
__global__ void k_build_psi(const double* __restrict__ xs, int64_t M, Geom g,
                            double* __restrict__ psi) {
  const int K = 2 * g.m + 1;
  const int64_t total = M * g.d * K;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    int t = (int)(q % K);
    int64_t r = q / K;
    int dim = (int)(r % g.d);
    int64_t i = r / g.d;
    double x = xs[dim * M + i];
    Stencil st = stencil(x, g.nd[dim], g.md);
    psi[q] = t < st.width ? dim_factor(g, dim, x, st.lo + t) * g.wscale[dim] : 0.0;
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

void bin_and_sort(const double* x_dev, int64_t M, const Geom& g, int maxsub, int ntiles,
                  int* perm, double* xs, int* tile_count, int* tile_start, int4** subs,
                  int* nsubs, cudaStream_t s) {
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

void build_psi(const double* xs, int64_t M, const Geom& g, double* psi, cudaStream_t s) {
  k_build_psi<<<blocks_for(M * g.d * (2 * g.m + 1), 256), 256, 0, s>>>(xs, M, g, psi);
  count_launch();
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
// transform.py:57-63 + :96-97: g[k mod n] = f_hat_k / |I_n| / phi_hat_0 /
// ... / phi_hat_{d-1} (division order kept), zero elsewhere.  One block row
// per grid line along the last dim (blockIdx.x = line, blockIdx.y = chunk).
struct DeconvGeom {
  int d;
  int N[MAX_D];
  int n[MAX_D];
  const double* col[MAX_D];  // phi_hat (times wscale) over k + N/2
  double grid_size;
};

template <typename R>
__global__ void k_deconv_pad(const cplx_t<R>* __restrict__ fhat, cplx_t<R>* __restrict__ grid,
                             DeconvGeom q) {
  const int dl = q.d - 1;
  const int nl = q.n[dl], Nl = q.N[dl];
  int64_t line = blockIdx.x;
  // decode the line's leading slots (dims 0..d-2), last dim slot from threads
  int kidx[MAX_D];
  bool inside = true;
  int64_t fl = 0, rem = line;
  int lead[MAX_D];
  for (int i = dl - 1; i >= 0; --i) { lead[i] = (int)(rem % q.n[i]); rem /= q.n[i]; }
  for (int i = 0; i < dl; ++i) {
    int sl = lead[i], Ni = q.N[i];
    int k = sl < Ni / 2 ? sl + Ni / 2 : (sl >= q.n[i] - Ni / 2 ? sl - q.n[i] + Ni / 2 : -1);
    if (k < 0) inside = false;
    kidx[i] = k;
    fl = fl * Ni + (k < 0 ? 0 : k);
  }
  cplx_t<R>* out = grid + line * nl;
  for (int sl = blockIdx.y * blockDim.x + threadIdx.x; sl < nl; sl += gridDim.y * blockDim.x) {
    cplx_t<R> v;
    v.x = 0;
    v.y = 0;
    int k = sl < Nl / 2 ? sl + Nl / 2 : (sl >= nl - Nl / 2 ? sl - nl + Nl / 2 : -1);
    if (inside && k >= 0) {
      cplx_t<R> a = fhat[fl * Nl + k];
      double re = (double)a.x / q.grid_size, im = (double)a.y / q.grid_size;
      for (int i = 0; i < dl; ++i) { double c = q.col[i][kidx[i]]; re /= c; im /= c; }
      double c = q.col[dl][k];
      re /= c;
      im /= c;
      v.x = (R)re;
      v.y = (R)im;
    }
    out[sl] = v;
  }
}

// transform.py:174-176: f_hat_k = g[k mod n] / |I_n| / prod phi_hat.
template <typename R>
__global__ void k_pack_deconv(const cplx_t<R>* __restrict__ grid, cplx_t<R>* __restrict__ fhat,
                              DeconvGeom q) {
  const int dl = q.d - 1;
  const int nl = q.n[dl], Nl = q.N[dl];
  int64_t line = blockIdx.x;  // line over N_0..N_{d-2}
  int kidx[MAX_D];
  int64_t gl = 0, rem = line;
  for (int i = dl - 1; i >= 0; --i) { kidx[i] = (int)(rem % q.N[i]); rem /= q.N[i]; }
  for (int i = 0; i < dl; ++i) {
    int k = kidx[i] - q.N[i] / 2;
    int sl = k < 0 ? k + q.n[i] : k;
    gl = gl * q.n[i] + sl;
  }
  for (int kl = blockIdx.y * blockDim.x + threadIdx.x; kl < Nl; kl += gridDim.y * blockDim.x) {
    int k = kl - Nl / 2;
    int sl = k < 0 ? k + nl : k;
    cplx_t<R> a = grid[gl * nl + sl];
    double re = (double)a.x / q.grid_size, im = (double)a.y / q.grid_size;
    for (int i = 0; i < dl; ++i) { double c = q.col[i][kidx[i]]; re /= c; im /= c; }
    double c = q.col[dl][kl];
    re /= c;
    im /= c;
    cplx_t<R> v;
    v.x = (R)re;
    v.y = (R)im;
    fhat[line * Nl + kl] = v;
  }
}

template <typename R>
void launch_deconv_pad(const void* fhat, void* grid, const DeconvGeom& q, cudaStream_t s) {
  int64_t lines = 1;
  for (int i = 0; i < q.d - 1; ++i) lines *= q.n[i];
  int nl = q.n[q.d - 1];
  dim3 grd((unsigned)lines, (unsigned)((nl + 255) / 256 > 65535 ? 65535 : (nl + 255) / 256));
  k_deconv_pad<R><<<grd, 256, 0, s>>>((const cplx_t<R>*)fhat, (cplx_t<R>*)grid, q);
  count_launch();
}

template <typename R>
void launch_pack_deconv(const void* grid, void* fhat, const DeconvGeom& q, cudaStream_t s) {
  int64_t lines = 1;
  for (int i = 0; i < q.d - 1; ++i) lines *= q.N[i];
  int Nl = q.N[q.d - 1];
  dim3 grd((unsigned)lines, (unsigned)((Nl + 255) / 256 > 65535 ? 65535 : (Nl + 255) / 256));
  k_pack_deconv<R><<<grd, 256, 0, s>>>((const cplx_t<R>*)grid, (cplx_t<R>*)fhat, q);
  count_launch();
}

// ---------------------------------------------------- tile halo helpers
template <int D>
__device__ __forceinline__ void tile_origin(const Geom& g, int tile, int* tc, int* org) {
  int t = tile;
#pragma unroll
  for (int i = D - 1; i >= 0; --i) {
    tc[i] = t % g.ntile[i];
    t /= g.ntile[i];
  }
#pragma unroll
  for (int i = 0; i < D; ++i) org[i] = tc[i] * g.T[i] - g.m;
}

// linear grid slot of halo cell idx (halo row-major, last dim fastest)
template <int D>
__device__ __forceinline__ int64_t halo_slot(const Geom& g, const int* org, int idx) {
  int a[D];
  int rem = idx;
#pragma unroll
  for (int i = D - 1; i >= 0; --i) {
    a[i] = rem % g.H[i];
    rem /= g.H[i];
  }
  int64_t lin = 0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    int s = org[i] + a[i];
    s = s % g.n[i];
    if (s < 0) s += g.n[i];
    lin = lin * g.n[i] + s;
  }
  return lin;
}

// Per-node stencil in halo coordinates: h = (cell slot - tile start) + m -
// (cell - lo); with cell - lo in {m-1, m} this stays inside [0, T + 2m].
template <int D>
__device__ __forceinline__ void node_stencil(const Geom& g, const int* tc, const double* x,
                                             int* h, int* W, int64_t* lo) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    Stencil st = stencil(x[i], g.nd[i], g.md);
    int64_t slot = floor_mod(st.cell, g.n[i]);
    h[i] = (int)(slot - (int64_t)tc[i] * g.T[i]) + g.m - (int)(st.cell - st.lo);
    W[i] = st.width;
    lo[i] = st.lo;
  }
}

template <typename R, int D>
__device__ __forceinline__ void node_weights(const Geom& g, int64_t i, const double* x,
                                             const int64_t* lo, const int* W, R* wb, int lane,
                                             int nlanes) {
  const int K = 2 * g.m + 1;
  for (int q = lane; q < D * K; q += nlanes) {
    int dim = q / K, t = q - dim * K;
    R v = 0;
    if (t < W[dim]) {
      if (g.mode == MODE_TENSOR)
        v = (R)g.psi[(i * D + dim) * K + t];
      else
        v = (R)(dim_factor(g, dim, x[dim], lo[dim] + t) * g.wscale[dim]);
    }
    wb[q] = v;
  }
}

__device__ __forceinline__ size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }

// ---------------------------------------------------------------- B (interp)
// kernels.py:122-197.  One CTA per subproblem (<= maxsub nodes of one tile):
// the tile's (T+2m+1)^d halo is staged in shared memory, then each warp takes
// one node at a time; lanes split the leading stencil dims and run along the
// contiguous last dim; a warp-shuffle reduction forms f_j.
template <typename R, int D>
__global__ void __launch_bounds__(256)
k_interp_tiled(const cplx_t<R>* __restrict__ grid, cplx_t<R>* __restrict__ fout,
               const double* __restrict__ xs, const int* __restrict__ perm,
               const int4* __restrict__ subs, Geom g) {
  using C = cplx_t<R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = 2 * g.m + 1;
  int hsz = 1;
#pragma unroll
  for (int i = 0; i < D; ++i) hsz *= g.H[i];
  C* halo = reinterpret_cast<C*>(smem_raw);
  R* wbuf = reinterpret_cast<R*>(smem_raw + align16((size_t)hsz * sizeof(C)));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  R* wmy = wbuf + warp * D * K;
  const int4 sp = subs[blockIdx.x];
  int tc[D], org[D];
  tile_origin<D>(g, sp.x, tc, org);
  for (int idx = threadIdx.x; idx < hsz; idx += blockDim.x) halo[idx] = grid[halo_slot<D>(g, org, idx)];
  __syncthreads();

  const int H1 = D > 1 ? g.H[1] : 1;
  const int H2 = D > 2 ? g.H[2] : 1;
  for (int i = sp.y + warp; i < sp.y + sp.z; i += nwarps) {
    double x[D];
#pragma unroll
    for (int dd = 0; dd < D; ++dd) x[dd] = xs[dd * g.M + i];
    int h[D], W[D];
    int64_t lo[D];
    node_stencil<D>(g, tc, x, h, W, lo);
    node_weights<R, D>(g, i, x, lo, W, wmy, lane, 32);
    __syncwarp();
    R are = 0, aim = 0;
    if constexpr (D == 1) {
      for (int t0 = lane; t0 < W[0]; t0 += 32) {
        C v = halo[h[0] + t0];
        R w = wmy[t0];
        are += w * v.x;
        aim += w * v.y;
      }
    } else if constexpr (D == 2) {
      for (int t0 = lane; t0 < W[0]; t0 += 32) {
        const C* row = halo + (h[0] + t0) * H1 + h[1];
        R sre = 0, sim = 0;
        for (int t1 = 0; t1 < W[D - 1]; ++t1) {
          C v = row[t1];
          R w = wmy[K + t1];
          sre += w * v.x;
          sim += w * v.y;
        }
        R w0 = wmy[t0];
        are += w0 * sre;
        aim += w0 * sim;
      }
    } else {
      const int P = W[0] * W[1];
      for (int p = lane; p < P; p += 32) {
        int t0 = p / W[1], t1 = p - t0 * W[1];
        const C* row = halo + ((h[0] + t0) * H1 + h[1] + t1) * H2 + h[D - 1];
        R sre = 0, sim = 0;
        for (int t2 = 0; t2 < W[D - 1]; ++t2) {
          C v = row[t2];
          R w = wmy[2 * K + t2];
          sre += w * v.x;
          sim += w * v.y;
        }
        R w01 = wmy[t0] * wmy[K + t1];
        are += w01 * sre;
        aim += w01 * sim;
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      are += __shfl_xor_sync(0xffffffffu, are, off);
      aim += __shfl_xor_sync(0xffffffffu, aim, off);
    }
    if (lane == 0) {
      C v;
      v.x = are;
      v.y = aim;
      fout[perm[i]] = v;
    }
    __syncwarp();
  }
}

// -------------------------------------------------------------- B^H (spread)
// kernels.py:209-401.  One CTA per subproblem accumulates into a shared-memory
// halo without atomics: halo rows along dim 0 are owned round-robin by "row
// units" (d=3: warps, d=2: half-warps, d=1: threads), so two units never touch
// the same cell -- the GPU analogue of the reference's slab ownership
// (kernels.py:13-17).  Node weights are computed once per batch and shared.
// The finished halo is added to the HBM grid with fp64 RED atomics.
constexpr int SPREAD_BATCH = 32;

template <typename R, int D>
__global__ void __launch_bounds__(256)
k_spread_tiled(cplx_t<R>* __restrict__ grid, const cplx_t<R>* __restrict__ fin,
               const double* __restrict__ xs, const int* __restrict__ perm,
               const int4* __restrict__ subs, Geom g) {
  using C = cplx_t<R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = 2 * g.m + 1;
  int hsz = 1;
#pragma unroll
  for (int i = 0; i < D; ++i) hsz *= g.H[i];
  C* halo = reinterpret_cast<C*>(smem_raw);
  size_t off = align16((size_t)hsz * sizeof(C));
  C* fval = reinterpret_cast<C*>(smem_raw + off);
  off += align16(SPREAD_BATCH * sizeof(C));
  int* hW = reinterpret_cast<int*>(smem_raw + off);  // [batch][2D]: h, W
  off += align16(SPREAD_BATCH * 2 * D * sizeof(int));
  R* wb = reinterpret_cast<R*>(smem_raw + off);      // [batch][D*K]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int4 sp = subs[blockIdx.x];
  int tc[D], org[D];
  tile_origin<D>(g, sp.x, tc, org);
  for (int idx = threadIdx.x; idx < hsz; idx += blockDim.x) {
    C z;
    z.x = 0;
    z.y = 0;
    halo[idx] = z;
  }
  const int H1 = D > 1 ? g.H[1] : 1;
  const int H2 = D > 2 ? g.H[2] : 1;
  const int end = sp.y + sp.z;
  for (int base = sp.y; base < end; base += SPREAD_BATCH) {
    const int nb = min(SPREAD_BATCH, end - base);
    for (int jb = warp; jb < nb; jb += nwarps) {
      const int i = base + jb;
      double x[D];
#pragma unroll
      for (int dd = 0; dd < D; ++dd) x[dd] = xs[dd * g.M + i];
      int h[D], W[D];
      int64_t lo[D];
      node_stencil<D>(g, tc, x, h, W, lo);
      node_weights<R, D>(g, i, x, lo, W, wb + jb * D * K, lane, 32);
      if (lane == 0) {
        fval[jb] = fin[perm[i]];
#pragma unroll
        for (int dd = 0; dd < D; ++dd) {
          hW[jb * 2 * D + dd] = h[dd];
          hW[jb * 2 * D + D + dd] = W[dd];
        }
      }
    }
    __syncthreads();
    if constexpr (D == 3) {
      const int unit = warp, U = nwarps;
      for (int jb = 0; jb < nb; ++jb) {
        const int* q = hW + jb * 2 * D;
        const int h0 = q[0], h1 = q[1], h2 = q[2], W0 = q[3], W1 = q[4], W2 = q[5];
        const R* w = wb + jb * D * K;
        const C f = fval[jb];
        const int P = W1 * W2;
        for (int a = h0 + ((unit - h0) % U + U) % U; a < h0 + W0; a += U) {
          R w0 = w[a - h0];
          R cre = f.x * w0, cim = f.y * w0;
          for (int p = lane; p < P; p += 32) {
            int t1 = p / W2, t2 = p - t1 * W2;
            R ww = w[K + t1] * w[2 * K + t2];
            C* cell = halo + (a * H1 + h1 + t1) * H2 + h2 + t2;
            C v = *cell;
            v.x += cre * ww;
            v.y += cim * ww;
            *cell = v;
          }
        }
        __syncwarp();
      }
    } else if constexpr (D == 2) {
      const int unit = threadIdx.x >> 4, U = blockDim.x >> 4, l16 = lane & 15;
      for (int jb = 0; jb < nb; ++jb) {
        const int* q = hW + jb * 2 * D;
        const int h0 = q[0], h1 = q[1], W0 = q[2], W1 = q[3];
        const R* w = wb + jb * D * K;
        const C f = fval[jb];
        for (int a = h0 + ((unit - h0) % U + U) % U; a < h0 + W0; a += U) {
          R w0 = w[a - h0];
          R cre = f.x * w0, cim = f.y * w0;
          for (int t1 = l16; t1 < W1; t1 += 16) {
            R ww = w[K + t1];
            C* cell = halo + a * H1 + h1 + t1;
            C v = *cell;
            v.x += cre * ww;
            v.y += cim * ww;
            *cell = v;
          }
        }
        __syncwarp();
      }
    } else {
      const int unit = threadIdx.x, U = blockDim.x;
      for (int jb = 0; jb < nb; ++jb) {
        const int* q = hW + jb * 2 * D;
        const int h0 = q[0], W0 = q[1];
        const R* w = wb + jb * D * K;
        const C f = fval[jb];
        for (int a = h0 + ((unit - h0) % U + U) % U; a < h0 + W0; a += U) {
          R w0 = w[a - h0];
          C v = halo[a];
          v.x += f.x * w0;
          v.y += f.y * w0;
          halo[a] = v;
        }
      }
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < hsz; idx += blockDim.x) {
    C v = halo[idx];
    if (v.x != (R)0 || v.y != (R)0) {
      int64_t lin = halo_slot<D>(g, org, idx);
      atomicAdd(&grid[lin].x, v.x);
      atomicAdd(&grid[lin].y, v.y);
    }
  }
}

size_t interp_smem(const Geom& g, int elem_bytes, int threads) {
  size_t hsz = 1;
  for (int i = 0; i < g.d; ++i) hsz *= g.H[i];
  return ((hsz * elem_bytes + 15) & ~(size_t)15) + (size_t)(threads / 32) * g.d * (2 * g.m + 1) * (elem_bytes / 2);
}

size_t spread_smem(const Geom& g, int elem_bytes) {
  size_t hsz = 1;
  for (int i = 0; i < g.d; ++i) hsz *= g.H[i];
  size_t off = (hsz * elem_bytes + 15) & ~(size_t)15;
  off += (SPREAD_BATCH * elem_bytes + 15) & ~(size_t)15;
  off += (SPREAD_BATCH * 2 * g.d * sizeof(int) + 15) & ~(size_t)15;
  off += (size_t)SPREAD_BATCH * g.d * (2 * g.m + 1) * (elem_bytes / 2);
  return off;
}

template <typename R, int D>
static void interp_launch(const void* grid, void* f, const double* xs, const int* perm,
                          const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  const int threads = 256;
  size_t smem = interp_smem(g, sizeof(cplx_t<R>), threads);
  auto kern = k_interp_tiled<R, D>;
  NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nsubs > 0) {
    kern<<<nsubs, threads, smem, s>>>((const cplx_t<R>*)grid, (cplx_t<R>*)f, xs, perm, subs, g);
    count_launch();
  }
}

template <typename R, int D>
static void spread_launch(void* grid, const void* f, const double* xs, const int* perm,
                          const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  const int threads = 256;
  size_t smem = spread_smem(g, sizeof(cplx_t<R>));
  auto kern = k_spread_tiled<R, D>;
  NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nsubs > 0) {
    kern<<<nsubs, threads, smem, s>>>((cplx_t<R>*)grid, (const cplx_t<R>*)f, xs, perm, subs, g);
    count_launch();
  }
}

void launch_interp(bool single, const void* grid, void* f, const double* xs, const int* perm,
                   const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  if (single) {
    if (g.d == 1) interp_launch<float, 1>(grid, f, xs, perm, subs, nsubs, g, s);
    else if (g.d == 2) interp_launch<float, 2>(grid, f, xs, perm, subs, nsubs, g, s);
    else interp_launch<float, 3>(grid, f, xs, perm, subs, nsubs, g, s);
  } else {
    if (g.d == 1) interp_launch<double, 1>(grid, f, xs, perm, subs, nsubs, g, s);
    else if (g.d == 2) interp_launch<double, 2>(grid, f, xs, perm, subs, nsubs, g, s);
    else interp_launch<double, 3>(grid, f, xs, perm, subs, nsubs, g, s);
  }
}

void launch_spread(bool single, void* grid, const void* f, const double* xs, const int* perm,
                   const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  if (single) {
    if (g.d == 1) spread_launch<float, 1>(grid, f, xs, perm, subs, nsubs, g, s);
    else if (g.d == 2) spread_launch<float, 2>(grid, f, xs, perm, subs, nsubs, g, s);
    else spread_launch<float, 3>(grid, f, xs, perm, subs, nsubs, g, s);
  } else {
    if (g.d == 1) spread_launch<double, 1>(grid, f, xs, perm, subs, nsubs, g, s);
    else if (g.d == 2) spread_launch<double, 2>(grid, f, xs, perm, subs, nsubs, g, s);
    else spread_launch<double, 3>(grid, f, xs, perm, subs, nsubs, g, s);
  }
}

void launch_deconv(bool single, const void* fhat, void* grid, const DeconvGeomH& qh, cudaStream_t s) {
  DeconvGeom q;
  q.d = qh.d;
  for (int i = 0; i < MAX_D; ++i) { q.N[i] = qh.N[i]; q.n[i] = qh.n[i]; q.col[i] = qh.col[i]; }
  q.grid_size = qh.grid_size;
  if (single) launch_deconv_pad<float>(fhat, grid, q, s);
  else launch_deconv_pad<double>(fhat, grid, q, s);
}

void launch_pack(bool single, const void* grid, void* fhat, const DeconvGeomH& qh, cudaStream_t s) {
  DeconvGeom q;
  q.d = qh.d;
  for (int i = 0; i < MAX_D; ++i) { q.N[i] = qh.N[i]; q.n[i] = qh.n[i]; q.col[i] = qh.col[i]; }
  q.grid_size = qh.grid_size;
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
