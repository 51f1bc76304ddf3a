// Plan lifecycle and transform orchestration for the B200 NFFT.
// Parameter validation follows Plan.__init__ (plan.py:138-186) check by check
// so the ABI reports the same error classes and codes as the reference.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "plan.h"

#include <cublas_v2.h>

namespace nfftk {

static std::string fmt_tuple(const std::vector<int>& v) {
  std::ostringstream os;
  os << "(";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) os << ", ";
    os << v[i];
  }
  if (v.size() == 1) os << ",";
  os << ")";
  return os.str();
}

static std::string fmt_double(double v) {
  // shortest round-trip representation, like Python's repr(float)
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eni") == std::string::npos) s += ".0";
  return s;
}

static std::string hexs(uint32_t v) {
  char buf[32];
  snprintf(buf, sizeof buf, "0x%x", v);
  return buf;
}

// ------------------------------------------------------- host window math
// window.py:38-53
double host_bessel_i0(double x) {
  double s = 1.0, t = 1.0, q = 0.25 * x * x;
  long j = 0;
  for (;;) {
    j += 1;
    t *= q / (double)(j * j);
    s += t;
    if (t < 1e-16 * s) return s;
  }
}

// window.py:56-72
double host_window(int code, double t, double n_i, double m, double b_i) {
  if (code == WINDOW_KB) {
    double nt = n_i * t;
    double u = m * m - nt * nt;
    if (u > 0.0) {
      double z = std::sqrt(u);
      return std::sinh(b_i * z) / (M_PI * z);
    }
    if (u < 0.0) {
      double z = std::sqrt(-u);
      return std::sin(b_i * z) / (M_PI * z);
    }
    return b_i / M_PI;
  }
  double nt = n_i * t;
  return std::exp(-nt * nt / b_i) / std::sqrt(M_PI * b_i);
}

// window.py:142-164 (phi_hat).  Returns 0 and the value, or 1 (the KB
// transform vanishes: b^2 < (2 pi k / n)^2) / 2 (value not positive).
int phi_hat_value(int code, int k, int n_i, int m, double b, double* out) {
  double val;
  if (code == WINDOW_KB) {
    double c = 2.0 * M_PI * k / n_i;
    double arg = b * b - c * c;
    if (arg < 0.0) return 1;
    val = host_bessel_i0(m * std::sqrt(arg)) / n_i;
  } else {
    double c = M_PI * k / n_i;
    val = std::exp(-b * c * c) / n_i;
  }
  *out = val;
  return val > 0.0 ? 0 : 2;
}

// window.py:101-111: b from sigma = n_i / N_i
double window_shape(int code, int N_i, int n_i, int m) {
  const double s = (double)n_i / (double)N_i;
  return code == WINDOW_KB ? M_PI * (2.0 - 1.0 / s) : 2.0 * s * m / ((2.0 * s - 1.0) * M_PI);
}

// checked strictly positive (WindowDegenerateError)
static double host_phi_hat(const Plan* p, int dim, int k) {
  double val = 0.0;
  switch (phi_hat_value(p->window, k, p->n[dim], p->m, p->b[dim], &val)) {
    case 1: fail(EK_WINDOW, "kaiserbessel transform vanishes at k=" + std::to_string(k));
    case 2: fail(EK_WINDOW, "window transform not positive at k=" + std::to_string(k));
    default: return val;
  }
}

std::vector<double> plan_phi_hut(const Plan* p, int dim) {
  // phi_hat_table(i, kmax=N_i/2) (window.py:166-171; plan.py:256)
  std::vector<double> out;
  int kmax = p->N[dim] / 2;
  for (int k = -kmax; k <= kmax; ++k) out.push_back(host_phi_hat(p, dim, k));
  return out;
}

// ------------------------------------------------------------ lifecycle
Plan::~Plan() {
  if (device >= 0) cudaSetDevice(device);
  if (fft_ready) cufftDestroy(fft);
  if (cublas) cublasDestroy((cublasHandle_t)cublas);
  cudaFree(x_dev);
  cudaFree(xs);
  cudaFree(perm);
  cudaFree(tile_count);
  cudaFree(subs);
  cudaFree(psi);
  cudaFree(rec);
  cudaFree(rrec);
  cudaFree(lut);
  cudaFree(cols);
  if (!grid_external) cudaFree(grid);
  cudaFree(gp);
  for (int i = 0; i < MAX_D; ++i) cudaFree(fft_tw[i]);
  cudaFree(sched);
  for (auto& h : hgraph)
    if (h.exec) cudaGraphExecDestroy(h.exec);
  cudaFree(fhat_dev);
  cudaFree(f_dev);
  cudaFree(f_sorted);
  if (fhat_pinned) cudaFreeHost(fhat_host); else free(fhat_host);
  if (f_pinned) cudaFreeHost(f_host); else free(f_host);
  for (auto& r : recs) { event_pool.push_back(r.a); event_pool.push_back(r.b); }
  for (auto e : event_pool) cudaEventDestroy(e);
  if (own_stream) cudaStreamDestroy(own_stream);
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// Tile edge per dim (powers of two).  d = 3: the smallest tile expected to
// hold >= 64 nodes whose halo fits 100 KB (two CTAs per SM), else the largest
// halo up to 190 KB (one CTA per SM, 16 warps) -- low node densities need big
// tiles to amortise the halo.  d = 2 / d = 1: the largest halo within
// 100 KB / 64 KB.  NFFTK_TILE overrides.
static void choose_tiles(Plan* p) {
  Geom& g = p->geom;
  const size_t KB = 1024;
  const size_t eb = p->elem_bytes();
  const double rho = (double)p->M / (double)p->grid_size;
  auto halo_bytes = [&](int T) {
    size_t h = 1;
    for (int i = 0; i < p->d; ++i) h *= (size_t)(std::min(T, p->n[i]) + 2 * p->m + 1);
    return h * eb;
  };
  int T = 0;
  if (p->d == 3) {
    for (int c : {4, 8, 16})
      if (rho * c * c * c >= 64.0 && halo_bytes(c) <= 100 * KB) { T = c; break; }
    if (!T)
      for (int c : {16, 8, 4, 2})
        if (halo_bytes(c) <= 190 * KB) { T = c; break; }
    if (!T) T = 2;
  } else if (p->d == 2) {
    // single-warp spread CTAs keep a private halo: small tiles
    for (int c : {16, 8, 4, 2})
      if (halo_bytes(c) <= 24 * KB) { T = c; break; }
    if (!T) T = 2;
  } else {
    for (int c = 512; c >= 2; c /= 2)
      if (halo_bytes(c) <= 16 * KB) { T = c; break; }
    if (!T) T = 2;
  }
  int force = env_int("NFFTK_TILE", 0);
  if (force > 0) T = force;
  // the padded extent must keep every padded index within one period of the
  // grid on either side (pad / fold wrap with one correction)
  auto fits = [&](int t) {
    for (int i = 0; i < p->d; ++i) {
      int ti = std::min(t, p->n[i]), nt = (p->n[i] + ti - 1) / ti;
      if (nt * ti + p->m + 2 > 2 * p->n[i]) return false;
    }
    return true;
  };
  while (T > 2 && !fits(T)) T /= 2;
  int Td[MAX_D];
  for (int i = 0; i < p->d; ++i) Td[i] = std::min(T, p->n[i]);
  // d = 2 register-resident spread: 32 halo rows (one warp) x (8 + 2m + 1)
  if (p->d == 2 && !force && p->m <= 8 && !getenv("NFFTK_NO_PIPE")) {
    const int t0 = 32 - (2 * p->m + 1), t1 = 8;
    auto fits1 = [&](int i, int ti) {
      int nt = (p->n[i] + ti - 1) / ti;
      return ti <= p->n[i] && nt * ti + p->m + 2 <= 2 * p->n[i];
    };
    if (fits1(0, t0) && fits1(1, t1)) {
      Td[0] = t0;
      Td[1] = t1;
    }
  }
  p->ntiles = 1;
  for (int i = 0; i < p->d; ++i) {
    g.T[i] = Td[i];
    g.H[i] = g.T[i] + 2 * p->m + 1;
    g.ntile[i] = (p->n[i] + g.T[i] - 1) / g.T[i];
    p->ntiles *= g.ntile[i];
  }
  // ghost-padded grid: pad m on the left, >= m+2 on the right (even length)
  for (int i = 0; i < p->d; ++i) {
    g.np[i] = g.ntile[i] * g.T[i] + 2 * p->m + 2;
  }
  g.HS = g.H[p->d - 1] + (eb == 8 ? 1 : 0);   // complex64 rows padded to 16-byte multiples
  g.nb_spread = 32;
  while (g.nb_spread > 4 && spread_smem_nb(g, (int)eb, g.nb_spread) > 220 * KB) g.nb_spread /= 2;
  g.nt_interp = interp_smem(g, (int)eb, 256) > 110 * KB ? 512 : 256;
  g.nt_interp = env_int("NFFTK_INTERP_THREADS", g.nt_interp);
  // nodes per subproblem (one CTA): at most 1024, and small enough that a
  // small plan still spreads over the SMs (C1: 4 tiles of 1024 nodes would
  // run on 4 CTAs)
  int ms = 1024;
  while (ms > 32 && (int64_t)ms * 4 * 148 > p->M) ms /= 2;
  p->maxsub = env_int("NFFTK_MAXSUB", ms);
  g.debug = env_int("NFFTK_DEBUG", 0);
  g.res = res_geometry(g, p->single) ? 1 : 0;
}

static void fill_geom(Plan* p) {
  Geom& g = p->geom;
  memset(&g, 0, sizeof g);
  g.d = p->d;
  g.m = p->m;
  g.md = (double)p->m;
  g.code = p->window;
  g.M = p->M;
  for (int i = 0; i < p->d && i < MAX_D; ++i) {
    g.n[i] = p->n[i];
    g.nd[i] = (double)p->n[i];
    g.b[i] = p->b[i];
    g.wscale[i] = p->wscale[i];
  }
  if (p->d <= MAX_D) choose_tiles(p);
}

Plan* plan_create(const std::vector<int>& N_in, int64_t M, const int* n_opt, const int* m_opt,
                  const uint32_t* f1_opt, const uint32_t* f2_opt, int window, bool single) {
  // validate_bandlimit (indexing.py:18-29)
  if (N_in.empty()) fail(EK_BANDLIMIT, "bandlimit vector is empty");
  for (int v : N_in)
    if (v < 2 || v % 2 != 0)
      fail(EK_BANDLIMIT, "bandlimit entries must be even and >= 2, got " + std::to_string(v));
  if (M < 1) fail(EK_NFFT, "node count must be >= 1, got " + std::to_string(M));
  if (window != WINDOW_KB && window != WINDOW_GAUSS)
    fail(EK_NFFT, "unknown window; use 'kaiserbessel' or 'gaussian'");
  if (M > 0x7fffffffLL) fail(EK_NFFT, "node count must fit in int32");
  Plan* p = new Plan();
  p->N = N_in;
  p->d = (int)N_in.size();
  p->M = M;
  p->window = window;
  p->single = single;
  try {
    // plan.py:144-167
    if (!n_opt) {
      for (int v : N_in) {
        int b = 0;
        while ((1 << b) < v) ++b;   // (v-1).bit_length()
        p->n.push_back(1 << (b + 1));
      }
      if (!m_opt)
        for (int& v : p->n)
          while (v < 2 * DEFAULT_CUTOFF + 2) v *= 2;
    } else {
      p->n.assign(n_opt, n_opt + p->d);
      for (int i = 0; i < p->d; ++i) {
        if (p->n[i] % 2 != 0)
          fail(EK_OVERSAMPLING, "FFT lengths must be even, got " + std::to_string(p->n[i]));
        if (p->n[i] <= p->N[i])
          fail(EK_OVERSAMPLING, "need n_i > N_i, got n=" + fmt_tuple(p->n) + " for N=" + fmt_tuple(p->N));
      }
    }
    int nmin = *std::min_element(p->n.begin(), p->n.end());
    // plan.py:168-176
    p->m = !m_opt ? std::min(DEFAULT_CUTOFF, (nmin - 1) / 2) : *m_opt;
    if (p->m < 1) fail(EK_CUTOFF, "cutoff must be >= 1, got " + std::to_string(p->m));
    if (2 * p->m + 1 > nmin)
      fail(EK_CUTOFF, "cutoff " + std::to_string(p->m) + " needs 2m+1 <= min(n) = " + std::to_string(nmin));
    if (p->m > 16) fail(EK_CUTOFF, "cutoff " + std::to_string(p->m) + " above the supported maximum 16");
    // plan.py:95-106, :177-178
    if (f1_opt) {
      uint32_t f1 = *f1_opt;
      uint32_t unknown = f1 & ~KNOWN_F1;
      if (unknown) fail(EK_FLAG, "unknown f1 bits: " + hexs(unknown));
      if (f1 & UNSUPPORTED_F1)
        fail(EK_UNSUPPORTED_FLAG, "fast Gaussian gridding flags (FG_PSI, PRE_FG_PSI) are not provided");
      p->f1 = f1;
    } else {
      p->f1 = PRE_PHI_HUT | PRE_PSI | NFFT_SORT_NODES | NOOP_F1 |
              (p->d > 1 ? NFFT_OMP_BLOCKWISE_ADJOINT : 0);
    }
    p->f2 = f2_opt ? *f2_opt : DEFAULT_F2;
    // WindowModel.make (window.py:91-112)
    for (int i = 0; i < p->d; ++i) {
      double s = (double)p->n[i] / (double)p->N[i];
      if (s <= 1.0) fail(EK_NFFT, "oversampling factor must exceed 1");
      if ((double)p->m / p->n[i] >= 0.5) fail(EK_NFFT, "window support m/n must be below 1/2");
      p->sigma.push_back(s);
      p->b.push_back(window_shape(window, p->N[i], p->n[i], p->m));
      // complex64 keeps window products in range by normalising by phi(0)
      p->wscale.push_back(single ? 1.0 / host_window(window, 0.0, p->n[i], p->m, p->b[i]) : 1.0);
    }
    p->num_freqs = 1;
    p->grid_size = 1;
    for (int i = 0; i < p->d; ++i) {
      p->num_freqs *= p->N[i];
      p->grid_size *= p->n[i];
    }
    if (p->d <= MAX_D && p->grid_size > (int64_t)0xffffffffLL)
      fail(EK_NFFT, "oversampled grid larger than 2^32 cells is not supported");
    if (cudaGetDevice(&p->device) != cudaSuccess) { p->device = 0; cudaGetLastError(); }
    fill_geom(p);
  } catch (...) {
    delete p;
    throw;
  }
  return p;
}

static void ensure_stream(Plan* p) {
  NFFTK_CUDA(cudaSetDevice(p->device));
  if (!p->own_stream) NFFTK_CUDA(cudaStreamCreateWithFlags(&p->own_stream, cudaStreamNonBlocking));
}

// ---------------------------------------------------------- phase events
struct PhaseScope {
  Plan* p;
  int ph;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  static cudaEvent_t take(Plan* p) {
    cudaEvent_t e;
    if (!p->event_pool.empty()) {
      e = p->event_pool.back();
      p->event_pool.pop_back();
    } else {
      NFFTK_CUDA(cudaEventCreate(&e));
    }
    return e;
  }
  PhaseScope(Plan* p_, int ph_, cudaStream_t s_) : p(p_), ph(ph_), s(s_) {
    if (!p->timing) return;
    a = take(p);
    b = take(p);
    cudaEventRecord(a, s);
  }
  ~PhaseScope() {
    if (!p->timing) return;
    cudaEventRecord(b, s);
    p->recs.push_back({ph, a, b});
  }
};

void plan_phase_times(Plan* p, double* ms, int64_t* calls, int nmax, int reset) {
  NFFTK_CUDA(cudaSetDevice(p->device));
  for (auto& r : p->recs) {
    NFFTK_CUDA(cudaEventSynchronize(r.b));
    float t = 0;
    cudaEventElapsedTime(&t, r.a, r.b);
    p->phase_ms[r.phase] += t;
    p->phase_calls[r.phase] += 1;
    p->event_pool.push_back(r.a);
    p->event_pool.push_back(r.b);
  }
  p->recs.clear();
  for (int i = 0; i < nmax && i < PH_COUNT; ++i) {
    if (ms) ms[i] = p->phase_ms[i];
    if (calls) calls[i] = p->phase_calls[i];
  }
  if (reset)
    for (int i = 0; i < PH_COUNT; ++i) { p->phase_ms[i] = 0; p->phase_calls[i] = 0; }
}

// ---------------------------------------------------------------- nodes
static void check_range_host(const Plan* p, const double* x) {
  int64_t total = p->M * p->d;
  for (int64_t q = 0; q < total; ++q) {
    double v = x[q];
    if (!(v >= -0.5 && v < 0.5))
      fail(EK_NODE_RANGE, "node " + std::to_string(q / p->d) + " coordinate " + fmt_double(v) +
                              " outside [-1/2, 1/2)");
  }
}

static void shape_check_x(const Plan* p, int64_t len) {
  if (len != p->M * p->d)
    fail(EK_SHAPE, "need " + std::to_string(p->M * p->d) + " coordinates (" + std::to_string(p->M) +
                       " nodes x " + std::to_string(p->d) + "), got " + std::to_string(len));
}

// Device part of set_nodes: tile binning + sort + sorted coordinates.
static void nodes_to_device(Plan* p, cudaStream_t s) {
  const int64_t M = p->M;
  if (!p->xs) NFFTK_CUDA(cudaMalloc(&p->xs, sizeof(double) * M * p->d));
  if (!p->perm) NFFTK_CUDA(cudaMalloc(&p->perm, sizeof(int) * (M + 4)));  // +4: aligned bulk copies
  if (!p->tile_count) {
    NFFTK_CUDA(cudaMalloc(&p->tile_count, sizeof(int) * (p->ntiles + 1) * 2));
    p->tile_start = p->tile_count + p->ntiles + 1;
  }
  bin_and_sort(p->x_dev, M, p->geom, p->maxsub, p->ntiles, p->perm, p->xs, p->tile_count,
               p->tile_start, &p->subs, &p->nsubs, s);
  p->width_sum = sum_widths(p->xs, M, p->geom, s);
  if (!p->rec) NFFTK_CUDA(cudaMalloc(&p->rec, sizeof(int4) * M));
  unsigned* nwide = nullptr;
  if (p->geom.res) {
    // +4: aligned bulk copies; the wide-node counter sits behind them
    if (!p->rrec) NFFTK_CUDA(cudaMalloc(&p->rrec, sizeof(unsigned) * (M + 8)));
    nwide = p->rrec + M + 4;
    NFFTK_CUDA(cudaMemsetAsync(p->rrec + M, 0, sizeof(unsigned) * 8, s));
  }
  build_recs(p->xs, M, p->geom, p->rec, p->geom.res ? p->rrec : nullptr, nwide, s);
  p->geom.rec = p->rec;
  p->geom.rrec = p->rrec;
  p->geom.nwide = 0;
  if (nwide) {
    unsigned cnt = 0;
    NFFTK_CUDA(cudaMemcpyAsync(&cnt, nwide, sizeof cnt, cudaMemcpyDeviceToHost, s));
    NFFTK_CUDA(cudaStreamSynchronize(s));
    p->geom.nwide = (int)std::min<unsigned>(cnt, 0x7fffffffu);
  }
}

// New nodes invalidate the tables; the PRE_PSI allocation itself is kept
// (precompute rebuilds it in place when the size matches): freeing and
// re-allocating tens of GiB cost ~0.2 s per set_nodes at C5.
static void invalidate_tables(Plan* p) {
  p->ready = false;
  p->geom.psi = nullptr;
}

void plan_set_nodes_host(Plan* p, const double* x, int64_t len) {
  ++p->gen;
  shape_check_x(p, len);
  check_range_host(p, x);
  if (p->d <= MAX_D) {
    // straight from the caller's buffer (the call blocks until the copy is
    // done); no host copy is kept -- the device holds the nodes
    ensure_stream(p);
    if (!p->x_dev) NFFTK_CUDA(cudaMalloc(&p->x_dev, sizeof(double) * p->M * p->d));
    NFFTK_CUDA(cudaMemcpyAsync(p->x_dev, x, sizeof(double) * p->M * p->d,
                               cudaMemcpyHostToDevice, p->own_stream));
    invalidate_tables(p);
    p->has_nodes = false;
    p->x_host.clear();
    p->x_host.shrink_to_fit();
    nodes_to_device(p, p->own_stream);
    NFFTK_CUDA(cudaStreamSynchronize(p->own_stream));
  } else {
    // d > 3 has no fast transform; the exact sums read the host copy
    std::vector<double> copy(x, x + p->M * p->d);
    invalidate_tables(p);
    p->x_host.swap(copy);
  }
  p->has_nodes = true;
}

void plan_set_nodes_device(Plan* p, const double* x, int64_t len, cudaStream_t s) {
  ++p->gen;
  shape_check_x(p, len);
  if (p->d > MAX_D) fail(EK_SHAPE, "fast transforms support d <= 3, got d=" + std::to_string(p->d));
  NFFTK_CUDA(cudaSetDevice(p->device));
  unsigned long long* bad = nullptr;
  unsigned long long first = ~0ULL;
  NFFTK_CUDA(cudaMallocAsync(&bad, sizeof first, s));
  NFFTK_CUDA(cudaMemcpyAsync(bad, &first, sizeof first, cudaMemcpyHostToDevice, s));
  launch_check_range(x, p->M * p->d, bad, s);
  NFFTK_CUDA(cudaMemcpyAsync(&first, bad, sizeof first, cudaMemcpyDeviceToHost, s));
  NFFTK_CUDA(cudaFreeAsync(bad, s));
  NFFTK_CUDA(cudaStreamSynchronize(s));
  if (first != ~0ULL) {
    double v = 0;
    NFFTK_CUDA(cudaMemcpy(&v, x + first, sizeof v, cudaMemcpyDeviceToHost));
    fail(EK_NODE_RANGE, "node " + std::to_string(first / p->d) + " coordinate " + fmt_double(v) +
                            " outside [-1/2, 1/2)");
  }
  if (!p->x_dev) NFFTK_CUDA(cudaMalloc(&p->x_dev, sizeof(double) * p->M * p->d));
  NFFTK_CUDA(cudaMemcpyAsync(p->x_dev, x, sizeof(double) * p->M * p->d, cudaMemcpyDeviceToDevice, s));
  invalidate_tables(p);
  p->has_nodes = false;
  p->x_host.clear();
  nodes_to_device(p, s);
  NFFTK_CUDA(cudaStreamSynchronize(s));
  p->has_nodes = true;
}

// ------------------------------------------------------------- precompute
static void build_tensor_map(Plan* p) {
  const Geom& g = p->geom;
  if (p->d == 1) { p->tmap_ready = true; return; }   // d = 1 uses a 1-D bulk copy
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    NFFTK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !encode) fail(EK_CUDA, "cuTensorMapEncodeTiled unavailable");
  }
  // complex128 = two FLOAT64 along the innermost dim; complex64 = one 8-byte element
  const int scale = p->single ? 1 : 2;
  const size_t eb = p->elem_bytes();
  cuuint64_t dims[3];
  cuuint64_t strides[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  int r = p->d;
  for (int i = 0; i < r; ++i) {
    dims[i] = (cuuint64_t)g.np[r - 1 - i];
    box[i] = (cuuint32_t)(i == 0 ? g.HS : g.H[r - 1 - i]);
  }
  dims[0] *= scale;
  box[0] *= scale;
  strides[0] = (cuuint64_t)g.np[r - 1] * eb;
  if (r == 3) strides[1] = (cuuint64_t)g.np[2] * g.np[1] * eb;
  CUresult res = encode((CUtensorMap*)p->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)r, p->gp, dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (res != CUDA_SUCCESS) fail(EK_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)res) + ")");
  p->tmap_ready = true;
}

static void ensure_cufft(Plan* p) {
  if (p->fft_ready) return;
  int nn[MAX_D];
  for (int i = 0; i < p->d; ++i) nn[i] = p->n[i];
  cufftResult r = cufftPlanMany(&p->fft, p->d, nn, nullptr, 1, 0, nullptr, 1, 0,
                                p->single ? CUFFT_C2C : CUFFT_Z2Z, 1);
  if (r != CUFFT_SUCCESS) fail(EK_CUDA, "cufftPlanMany failed (" + std::to_string((int)r) + ")");
  p->fft_ready = true;
}

static void ensure_grid(Plan* p) {
  if (!p->grid) NFFTK_CUDA(cudaMalloc(&p->grid, p->elem_bytes() * p->grid_size));
  if (!p->sched) {
    NFFTK_CUDA(cudaMalloc(&p->sched, sizeof(unsigned) * SCHED_SLOTS));
    NFFTK_CUDA(cudaMemset(p->sched, 0, sizeof(unsigned) * SCHED_SLOTS));
  }
  p->geom.sched = getenv("NFFTK_STATIC_SCHED") ? nullptr : p->sched;
  if (!p->gp) {
    size_t cells = 1;
    for (int i = 0; i < p->d; ++i) cells *= (size_t)p->geom.np[i];
    p->gp_bytes = cells * p->elem_bytes();
    NFFTK_CUDA(cudaMalloc(&p->gp, p->gp_bytes));
    p->pq.d = p->d;
    p->pq.m = p->m;
    for (int i = 0; i < p->d; ++i) {
      p->pq.n[i] = p->n[i];
      p->pq.np[i] = p->geom.np[i];
    }
  }
  if (!p->tmap_ready) build_tensor_map(p);
  // pruned F / F^H (fft.cu) where the geometry allows it and its two
  // intermediate arrays fit the dense grid buffer (the trafo's scratch)
  p->fft3 = p->d <= MAX_D && fft3_supported(p->d, p->n.data(), p->N.data(), p->single);
  if (p->fft3) {
    p->fq.d = p->d;
    for (int i = 0; i < p->d; ++i) {
      p->fq.N[i] = p->N[i];
      p->fq.n[i] = p->n[i];
      p->fq.np[i] = p->geom.np[i];
    }
    if (fft3_scratch_elems(p->fq) > (size_t)p->grid_size) p->fft3 = false;
  }
  if (p->fft3) {
    p->fq.m = p->m;
    p->fq.grid_size = (double)p->grid_size;
    for (int i = 0; i < p->d; ++i) {
      if (!p->fft_tw[i]) {
        std::vector<unsigned char> tw;
        fft3_twiddles(p->n[i], p->single, tw);
        NFFTK_CUDA(cudaMalloc(&p->fft_tw[i], tw.size()));
        NFFTK_CUDA(cudaMemcpy(p->fft_tw[i], tw.data(), tw.size(), cudaMemcpyHostToDevice));
      }
      p->fq.tw[i] = p->fft_tw[i];
      p->fq.icol[i] = p->dq.icol[i];
    }
  } else {
    ensure_cufft(p);
  }
}

void plan_precompute(Plan* p, cudaStream_t s) {
  if (!p->has_nodes) fail(EK_STATE, "set nodes before precompute()");
  ++p->gen;
  if (p->d > MAX_D) {
    // plan.py:278-279: full tables are limited to d <= 3; others only need host tables
    if (p->f1 & PRE_FULL_PSI)
      fail(EK_NFFT, "full window tables support d <= 3, got d=" + std::to_string(p->d));
    for (int i = 0; i < p->d; ++i) plan_phi_hut(p, i);
    p->ready = true;
    return;
  }
  NFFTK_CUDA(cudaSetDevice(p->device));
  // PRE_PHI_HUT: deconvolution columns over k = -N/2 .. N/2-1 (transform.py:44-54);
  // the device always keeps them (their cost is negligible).
  std::vector<double> cols;
  for (int i = 0; i < p->d; ++i) {
    std::vector<double> c = plan_deconv_cols(p, i);
    cols.insert(cols.end(), c.begin(), c.end());
  }
  if (!p->cols) NFFTK_CUDA(cudaMalloc(&p->cols, sizeof(double) * cols.size()));
  NFFTK_CUDA(cudaMemcpyAsync(p->cols, cols.data(), sizeof(double) * cols.size(),
                             cudaMemcpyHostToDevice, s));
  p->dq.d = p->d;
  p->dq.grid_size = (double)p->grid_size;
  size_t off = 0;
  for (int i = 0; i < p->d; ++i) {
    p->dq.N[i] = p->N[i];
    p->dq.n[i] = p->n[i];
    p->dq.icol[i] = p->cols + off;
    off += p->N[i];
  }
  // factor mode precedence PSI > LUT > DIRECT (transform.py:72-80)
  int mode = MODE_DIRECT;
  if (p->f1 & (PRE_PSI | PRE_FULL_PSI)) mode = MODE_TENSOR;
  else if (p->f1 & PRE_LIN_PSI) mode = MODE_LUT;
  if (p->psi_policy >= 0 && !(mode == MODE_LUT)) mode = p->psi_policy;
  if (mode == MODE_LUT || (p->f1 & PRE_LIN_PSI)) {
    // plan.py:285-295 -- LUT built on the host with the reference's formula
    std::vector<double> lut((size_t)p->d * (LUT_SIZE + 1));
    for (int i = 0; i < p->d; ++i) {
      double h = ((double)p->m / p->n[i]) / LUT_SIZE;
      for (int t = 0; t <= LUT_SIZE; ++t)
        lut[(size_t)i * (LUT_SIZE + 1) + t] = host_window(p->window, t * h, p->n[i], p->m, p->b[i]);
      p->geom.lut_step[i] = LUT_SIZE / ((double)p->m / p->n[i]);
    }
    if (!p->lut) NFFTK_CUDA(cudaMalloc(&p->lut, sizeof(double) * lut.size()));
    NFFTK_CUDA(cudaMemcpyAsync(p->lut, lut.data(), sizeof(double) * lut.size(),
                               cudaMemcpyHostToDevice, s));
    p->geom.lut = p->lut;
  }
  p->geom.mode = MODE_DIRECT;  // psi table itself is built from exact factors
  p->geom.psi = nullptr;
  p->geom.psi_pad = 0;
  p->geom.psi_f32 = 0;
  p->geom.pr = psi_row(p->d, 2 * p->m + 1);
  if (mode == MODE_TENSOR) {
    const int K = 2 * p->m + 1;
    p->geom.psi_pad = p->d == 3 && pipe_geometry(p->geom) ? (pipe_sten3(p->single, p->m) ? 2 : 1) : 0;
    const int pad_count = p->geom.psi_pad == 2 ? sten3_count(K) : psi_row_halo(p->d, p->geom.H, K);
    p->geom.pr = p->geom.psi_pad ? psi_row_pad<double>(pad_count) : psi_row(p->d, K);
    // c64 plans on the pipelined geometries (only the pipelined kernels read
    // the table there) keep fp32 factor rows: half the bytes, no per-FMA
    // fp64 -> fp32 conversions
    if (p->single && pipe_geometry(p->geom)) {
      p->geom.psi_f32 = 1;
      p->geom.pr = psi_row_pad<float>(p->geom.psi_pad ? pad_count : p->d * K);
    }
    const size_t esz = p->geom.psi_f32 ? sizeof(float) : sizeof(double);
    // psi_count counts doubles of storage
    size_t count = ((size_t)p->M * p->geom.pr * esz + sizeof(double) - 1) / sizeof(double);
    if (p->psi && count != p->psi_count) {
      cudaFree(p->psi);
      p->psi = nullptr;
    }
    p->psi_count = count;
    if (!p->psi) NFFTK_CUDA(cudaMalloc(&p->psi, sizeof(double) * count));
    build_psi(p->xs, p->M, p->geom, p->psi, s);
    p->geom.psi = p->psi;
  }
  p->geom.mode = mode;
  p->mode = mode;
  p->geom.dense_flush = spread_dense_ok(p->geom, p->elem_bytes()) ? 1 : 0;
  ensure_grid(p);
  NFFTK_CUDA(cudaStreamSynchronize(s));
  p->ready = true;
}

// ------------------------------------------------------------- transforms
static void require_ready(const Plan* p) {
  // transform.py:85-89
  if (!p->has_nodes) fail(EK_STATE, "plan has no nodes; call set_nodes() first");
  if (!p->ready) fail(EK_STATE, "plan not precomputed; call precompute() first");
  if (p->d > MAX_D)
    fail(EK_SHAPE, "fast transforms support d <= 3, got d=" + std::to_string(p->d));
}

static void count_evals(Plan* p) {
  int64_t e = p->mode == MODE_DIRECT ? (int64_t)p->width_sum : 0;
  p->window_evals_last = e;
  p->window_evals_total += e;
}

static void exec_fft(Plan* p, int dir, cudaStream_t s) {
  NFFTK_CUDA(cudaGetLastError());
  ensure_cufft(p);
  if (cufftSetStream(p->fft, s) != CUFFT_SUCCESS) fail(EK_CUDA, "cufftSetStream failed");
  cufftResult r = p->single ? cufftExecC2C(p->fft, (cufftComplex*)p->grid, (cufftComplex*)p->grid, dir)
                            : cufftExecZ2Z(p->fft, (cufftDoubleComplex*)p->grid,
                                           (cufftDoubleComplex*)p->grid, dir);
  if (r != CUFFT_SUCCESS) fail(EK_CUDA, "cufftExec failed (" + std::to_string((int)r) + ")");
}

// B alone (kernels.py:122-197): samples at the plan's nodes from the dense
// n-grid already in p->grid (the multi-GPU trafo fills a bound grid with a
// distributed F first).
void plan_interp_device(Plan* p, void* f, cudaStream_t s) {
  require_ready(p);
  NFFTK_CUDA(cudaSetDevice(p->device));
  { PhaseScope ps(p, PH_PAD, s); launch_pad(p->single, p->grid, p->gp, p->pq, s); }
  { PhaseScope ps(p, PH_INTERP, s);
    launch_interp(p->single, p->tmap, p->gp, f, p->xs, p->perm, p->subs, p->nsubs, p->geom, s); }
  NFFTK_CUDA(cudaGetLastError());
  count_evals(p);
}

void plan_trafo_device(Plan* p, const void* fhat, void* f, cudaStream_t s) {
  require_ready(p);
  NFFTK_CUDA(cudaSetDevice(p->device));
  if (p->fft3) {
    // D, F and the ghost padding in three pruned passes: f_hat -> (scratch in
    // the dense grid buffer) -> the padded grid the gather reads
    { PhaseScope ps(p, PH_FFT_FWD, s); fft3_forward(p->single, fhat, p->grid, p->gp, true, p->fq, s); }
    { PhaseScope ps(p, PH_INTERP, s);
      launch_interp(p->single, p->tmap, p->gp, f, p->xs, p->perm, p->subs, p->nsubs, p->geom, s); }
    NFFTK_CUDA(cudaGetLastError());
    count_evals(p);
    return;
  }
  { PhaseScope ps(p, PH_DECONV, s); launch_deconv(p->single, fhat, p->grid, p->dq, s); }
  { PhaseScope ps(p, PH_FFT_FWD, s); exec_fft(p, CUFFT_FORWARD, s); }
  plan_interp_device(p, f, s);
}

// Deconvolution column of dim i as the kernels apply it: 1 / (phi_hat_i(k)
// * wscale_i) for k = -N_i/2 .. N_i/2 - 1 (transform.py:44-54; wscale is the
// complex64 window normalisation, 1 for complex128).
std::vector<double> plan_deconv_cols(const Plan* p, int dim) {
  std::vector<double> t = plan_phi_hut(p, dim), out;
  for (int k = 0; k < p->N[dim]; ++k) out.push_back(1.0 / (t[k] * p->wscale[dim]));
  return out;
}

void plan_spread_device(Plan* p, const void* f, cudaStream_t s) {
  require_ready(p);
  NFFTK_CUDA(cudaSetDevice(p->device));
  // dense flush: the pipelined spread reduces into the dense grid directly
  // (periodic wrap per halo row), so there is no ghost-padded grid to fold
  const bool dense = p->geom.dense_flush != 0;
  void* target = dense ? p->grid : p->gp;
  { PhaseScope ps(p, PH_ZERO, s);
    NFFTK_CUDA(cudaMemsetAsync(target, 0, dense ? p->elem_bytes() * (size_t)p->grid_size : p->gp_bytes, s)); }
  // (the residue spread and the d = 2 pipelined spread gather the samples themselves: no sorted copy)
  if (!spread_gathers(p->geom, p->single)) {
    if (!p->f_sorted) NFFTK_CUDA(cudaMalloc(&p->f_sorted, p->elem_bytes() * (p->M + 2)));  // +2: aligned bulk copies
    PhaseScope ps(p, PH_PERMUTE, s); launch_permute(p->single, f, p->perm, p->M, p->f_sorted, s); }
  { PhaseScope ps(p, PH_SPREAD, s);
    launch_spread(p->single, target, f, p->f_sorted, p->xs, p->perm, p->subs, p->nsubs, p->geom, s); }
  if (!dense) { PhaseScope ps(p, PH_FOLD, s); launch_fold(p->single, p->gp, p->grid, p->pq, s); }
  NFFTK_CUDA(cudaGetLastError());
  count_evals(p);
}

void plan_adjoint_finish_device(Plan* p, void* fhat, cudaStream_t s) {
  require_ready(p);
  NFFTK_CUDA(cudaSetDevice(p->device));
  if (p->fft3) {
    // F^H, the pack and D^H in three pruned passes; the padded grid buffer
    // (idle during the adjoint) and then the dense grid itself are scratch
    { PhaseScope ps(p, PH_FFT_INV, s); fft3_inverse(p->single, p->grid, p->gp, p->grid, fhat, p->fq, s); }
    NFFTK_CUDA(cudaGetLastError());
    return;
  }
  { PhaseScope ps(p, PH_FFT_INV, s); exec_fft(p, CUFFT_INVERSE, s); }
  { PhaseScope ps(p, PH_PACK, s); launch_pack(p->single, p->grid, fhat, p->dq, s); }
  NFFTK_CUDA(cudaGetLastError());
}

void plan_adjoint_device(Plan* p, const void* f, void* fhat, cudaStream_t s) {
  plan_spread_device(p, f, s);
  plan_adjoint_finish_device(p, fhat, s);
}

static void ensure_io(Plan* p) {
  if (!p->fhat_dev) NFFTK_CUDA(cudaMalloc(&p->fhat_dev, p->elem_bytes() * p->num_freqs));
  if (!p->f_dev) NFFTK_CUDA(cudaMalloc(&p->f_dev, p->elem_bytes() * p->M));
}

static bool is_pinned(const void* h) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// nfftk_set_fhat / nfftk_set_f (cabi.py:149-160 copy into the library buffer):
// the copy into the pinned library buffer goes chunk by chunk, each chunk
// followed by its host-to-device copy on the plan's stream, so the PCIe
// transfer runs under the host copy and the transform that follows finds its
// input on the device.  complex128 plans with pinned buffers only.
bool plan_host_upload_begin(Plan* p, bool fhat) {
  (fhat ? p->fhat_dev_cur : p->f_dev_cur) = false;
  if (p->single || p->d > MAX_D || getenv("NFFTK_NO_EAGER_UPLOAD")) return false;
  if (!(fhat ? p->fhat_pinned : p->f_pinned)) return false;
  NFFTK_CUDA(cudaSetDevice(p->device));
  ensure_stream(p);
  ensure_io(p);
  NFFTK_CUDA(cudaStreamSynchronize(p->own_stream));  // an earlier upload still reads the buffer
  return true;
}

void plan_host_upload_chunk(Plan* p, bool fhat, size_t off, size_t bytes) {
  char* dev = (char*)(fhat ? p->fhat_dev : p->f_dev);
  const char* host = (const char*)(fhat ? p->fhat_host : p->f_host);
  NFFTK_CUDA(cudaMemcpyAsync(dev + off, host + off, bytes, cudaMemcpyHostToDevice, p->own_stream));
}

void plan_host_upload_end(Plan* p, bool fhat) { (fhat ? p->fhat_dev_cur : p->f_dev_cur) = true; }

static void trafo_host_body(Plan* p, const void* fhat, void* f, cudaStream_t s) {
  if (!(fhat == p->fhat_host && p->fhat_dev_cur)) {
    PhaseScope ps(p, PH_H2D, s);
    NFFTK_CUDA(cudaMemcpyAsync(p->fhat_dev, fhat, p->elem_bytes() * p->num_freqs,
                               cudaMemcpyHostToDevice, s)); }
  plan_trafo_device(p, p->fhat_dev, p->f_dev, s);
  { PhaseScope ps(p, PH_D2H, s);
    NFFTK_CUDA(cudaMemcpyAsync(f, p->f_dev, p->elem_bytes() * p->M, cudaMemcpyDeviceToHost, s)); }
}

static void adjoint_host_body(Plan* p, const void* f, void* fhat, cudaStream_t s) {
  if (!(f == p->f_host && p->f_dev_cur)) {
    PhaseScope ps(p, PH_H2D, s);
    NFFTK_CUDA(cudaMemcpyAsync(p->f_dev, f, p->elem_bytes() * p->M, cudaMemcpyHostToDevice, s)); }
  plan_adjoint_device(p, p->f_dev, p->fhat_dev, s);
  { PhaseScope ps(p, PH_D2H, s);
    NFFTK_CUDA(cudaMemcpyAsync(fhat, p->fhat_dev, p->elem_bytes() * p->num_freqs,
                               cudaMemcpyDeviceToHost, s)); }
}

// Runs body eagerly, or through the plan's captured graph for this
// direction: the first call with a given (in, out, plan state) runs eagerly
// (one-time allocations and attribute setup happen there), the second
// captures and launches the graph, later ones only launch it.  Pinned host
// buffers only (a graph's memcpy nodes need them); phase timing runs eagerly.
template <typename Body>
static void host_call(Plan* p, int dir, const void* in, void* out, Body body) {
  cudaStream_t s = p->own_stream;
  Plan::HostGraph& h = p->hgraph[dir];
  // whether this call's input is already on the device (set_fhat / set_f
  // uploaded it, or it is the previous transform's result): part of the key,
  // a captured graph either contains the host-to-device copy or does not
  const bool skip = dir == 0 ? (in == p->fhat_host && p->fhat_dev_cur) : (in == p->f_host && p->f_dev_cur);
  const bool same = h.in == in && h.out == out && h.gen == p->gen && h.skip_h2d == skip;
  if (!same) {
    if (h.exec) cudaGraphExecDestroy(h.exec);
    h = Plan::HostGraph();
    h.in = in;
    h.out = out;
    h.gen = p->gen;
    h.skip_h2d = skip;
  }
  const bool usable = !p->graphs_off && !p->timing && !getenv("NFFTK_NO_HOST_GRAPH") &&
                      is_pinned(in) && is_pinned(out);
  bool captured_now = false;
  if (usable && !h.exec && h.seen >= 1) {
    const unsigned long long l0 = launch_count();
    cudaGraph_t graph = nullptr;
    NFFTK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      body(s);
    } catch (...) {
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      throw;
    }
    NFFTK_CUDA(cudaStreamEndCapture(s, &graph));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {  // keep the eager launches for this plan
      cudaGetLastError();
      p->graphs_off = true;
    } else {
      h.exec = exec;
      h.launches = launch_count() - l0;
      add_launches(0ull - h.launches);  // the capture itself launched nothing
      captured_now = true;              // ... but body() already counted this call's evals
    }
  }
  ++h.seen;
  if (usable && h.exec) {
    NFFTK_CUDA(cudaGraphLaunch(h.exec, s));
    add_launches(h.launches);
    if (!captured_now) count_evals(p);  // the host-side update a replay skips
  } else {
    body(s);
  }
  NFFTK_CUDA(cudaStreamSynchronize(s));
}

void plan_trafo_host(Plan* p, const void* fhat, void* f) {
  require_ready(p);
  ensure_stream(p);
  ensure_io(p);
  host_call(p, 0, fhat, f, [&](cudaStream_t s) { trafo_host_body(p, fhat, f, s); });
  // f_dev holds the samples just copied to f; fhat_dev still holds the input
  p->f_dev_cur = f == p->f_host;
  p->fhat_dev_cur = fhat == p->fhat_host;
}

void plan_adjoint_host(Plan* p, const void* f, void* fhat) {
  require_ready(p);
  ensure_stream(p);
  ensure_io(p);
  if (!p->f_sorted) NFFTK_CUDA(cudaMalloc(&p->f_sorted, p->elem_bytes() * (p->M + 2)));
  host_call(p, 1, f, fhat, [&](cudaStream_t s) { adjoint_host_body(p, f, fhat, s); });
  p->fhat_dev_cur = fhat == p->fhat_host;
  p->f_dev_cur = f == p->f_host;
}

void plan_node_order(Plan* p, int64_t* out) {
  if (!p->has_nodes) fail(EK_STATE, "plan has no nodes; call set_nodes() first");
  if (p->d > MAX_D) fail(EK_SHAPE, "node order on the device supports d <= 3");
  ensure_stream(p);
  int* order = nullptr;
  NFFTK_CUDA(cudaMalloc(&order, sizeof(int) * p->M));
  lex_order(p->x_dev, p->M, p->geom, order, p->own_stream);
  std::vector<int> tmp(p->M);
  NFFTK_CUDA(cudaMemcpyAsync(tmp.data(), order, sizeof(int) * p->M, cudaMemcpyDeviceToHost,
                             p->own_stream));
  NFFTK_CUDA(cudaStreamSynchronize(p->own_stream));
  cudaFree(order);
  for (int64_t i = 0; i < p->M; ++i) out[i] = tmp[i];
}

// PrecomputeTables.psi / psi_full_* (plan.py:109-121) in the reference
// layout, natural node order, computed on the device and copied to the
// caller's host arrays; vals / idx / counts may be null (psi only).
void plan_psi_tables(Plan* p, double* psi, double* vals, int64_t* idx, int64_t* counts) {
  if (!p->has_nodes) fail(EK_STATE, "plan has no nodes; call set_nodes() first");
  if (p->d > MAX_D) fail(EK_NFFT, "full window tables support d <= 3, got d=" + std::to_string(p->d));
  ensure_stream(p);
  cudaStream_t s = p->own_stream;
  const int K = 2 * p->m + 1;
  int64_t P = 1;
  for (int i = 0; i < p->d; ++i) P *= K;
  const size_t npsi = (size_t)p->M * p->d * K, nfull = vals ? (size_t)p->M * P : 0;
  double *dpsi = nullptr, *dvals = nullptr;
  int64_t *didx = nullptr, *dcnt = nullptr;
  NFFTK_CUDA(cudaMallocAsync(&dpsi, sizeof(double) * npsi, s));
  if (vals) {
    NFFTK_CUDA(cudaMallocAsync(&dvals, sizeof(double) * nfull, s));
    NFFTK_CUDA(cudaMallocAsync(&didx, sizeof(int64_t) * nfull, s));
    NFFTK_CUDA(cudaMallocAsync(&dcnt, sizeof(int64_t) * p->M, s));
  }
  Geom g = p->geom;
  g.wscale[0] = g.wscale[1] = g.wscale[2] = 1.0;
  psi_reference(p->x_dev, p->M, g, dpsi, dvals, didx, dcnt, s);
  if (psi) NFFTK_CUDA(cudaMemcpyAsync(psi, dpsi, sizeof(double) * npsi, cudaMemcpyDeviceToHost, s));
  if (vals) {
    NFFTK_CUDA(cudaMemcpyAsync(vals, dvals, sizeof(double) * nfull, cudaMemcpyDeviceToHost, s));
    NFFTK_CUDA(cudaMemcpyAsync(idx, didx, sizeof(int64_t) * nfull, cudaMemcpyDeviceToHost, s));
    NFFTK_CUDA(cudaMemcpyAsync(counts, dcnt, sizeof(int64_t) * p->M, cudaMemcpyDeviceToHost, s));
  }
  NFFTK_CUDA(cudaFreeAsync(dpsi, s));
  if (vals) {
    NFFTK_CUDA(cudaFreeAsync(dvals, s));
    NFFTK_CUDA(cudaFreeAsync(didx, s));
    NFFTK_CUDA(cudaFreeAsync(dcnt, s));
  }
  NFFTK_CUDA(cudaStreamSynchronize(s));
}

// PrecomputeTables.lut / lut_steps (plan.py:285-295) of a PRE_LIN_PSI plan
void plan_lut_tables(Plan* p, double* lut, double* steps) {
  if (!p->ready || !p->lut) fail(EK_STATE, "no PRE_LIN_PSI table; set the flag and call precompute()");
  NFFTK_CUDA(cudaSetDevice(p->device));
  NFFTK_CUDA(cudaMemcpy(lut, p->lut, sizeof(double) * p->d * (LUT_SIZE + 1), cudaMemcpyDeviceToHost));
  for (int i = 0; i < p->d; ++i) steps[i] = p->geom.lut_step[i];
}

void plan_bind_grid(Plan* p, void* dev, int64_t bytes) {
  if (bytes < (int64_t)(p->elem_bytes() * p->grid_size))
    fail(EK_SHAPE, "grid workspace needs " + std::to_string(p->elem_bytes() * p->grid_size) + " bytes");
  NFFTK_CUDA(cudaSetDevice(p->device));
  if (p->grid && !p->grid_external) cudaFree(p->grid);
  p->grid = dev;
  p->grid_external = true;
  ++p->gen;
}

}  // namespace nfftk
