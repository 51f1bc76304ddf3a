// extern "C" boundary of libnfftk.so.
//
// The 13 reference symbols (include/nfftk.h, reference pkg/include/nfftk.h:22-59)
// keep the semantics of the reference's flat handle API (cabi.py:1-245 behind
// the cffi shim abi.py:162-275): opaque int32 handles in a locked registry,
// library-owned zero-initialised interleaved-complex buffers, 0 / -1 / -2 /
// -3 / -9 return codes, a per-handle last error.  Everything else is an
// nfftk_* extension for the B200 build (device pointers, streams, dtype,
// phase timing, multi-GPU grid binding).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include <omp.h>

#include "plan.h"

using namespace nfftk;

namespace {

// One handle.  `mu` serialises every call on the handle: the reference
// documents that a plan may be shared by concurrent callers (serialised by
// the GIL there); here the transforms share per-plan device scratch (grid,
// staging buffers, ticket counters, captured graphs), so a second thread on
// the same handle waits instead of interleaving with the first.
struct Entry {
  Plan* plan = nullptr;
  int err_code = 0;
  int err_kind = 0;
  std::string err_msg;
  std::mutex mu;
};

std::mutex g_lock;
std::unordered_map<int32_t, std::shared_ptr<Entry>> g_registry;
int32_t g_next_handle = 1;
int64_t g_live_buffers = 0;
thread_local int g_create_kind = 0;
thread_local std::string g_create_msg;
const char* const ABI_VERSION = "0.1.0";
const char* const EXT_VERSION = "b200-0.1.0";

std::shared_ptr<Entry> lookup_shared(int32_t h) {
  std::lock_guard<std::mutex> g(g_lock);
  auto it = g_registry.find(h);
  return it == g_registry.end() ? nullptr : it->second;
}

// A looked-up handle, locked for the duration of one ABI call.  Converts to
// nullptr for an unknown (or concurrently destroyed) handle.
class EntryLock {
 public:
  explicit EntryLock(int32_t h) : e_(lookup_shared(h)) {
    if (e_) lk_ = std::unique_lock<std::mutex>(e_->mu);
  }
  operator Entry*() const { return e_ && e_->plan ? e_.get() : nullptr; }
  Entry* operator->() const { return e_.get(); }

 private:
  std::shared_ptr<Entry> e_;
  std::unique_lock<std::mutex> lk_;
};

int32_t store(Entry* e, int kind, const std::string& msg) {
  e->err_kind = kind;
  e->err_code = abi_code(kind);
  e->err_msg = msg;
  return e->err_code;
}

template <typename F>
int32_t guarded(Entry* e, F&& fn) {
  try {
    fn();
    e->err_code = 0;
    e->err_kind = 0;
    return 0;
  } catch (const Error& err) {
    return store(e, err.kind, err.what());
  } catch (const std::bad_alloc&) {
    return store(e, EK_NFFT, "host allocation failed");
  } catch (const std::exception& err) {
    return store(e, EK_NFFT, err.what());
  }
}

int32_t do_create(const int32_t* bandlimits, int32_t rank, int32_t node_count,
                  const int32_t* n, const int* m, const uint32_t* f1, const uint32_t* f2, int window,
                  bool single) {
  g_create_kind = 0;
  g_create_msg.clear();
  if (rank < 1 || !bandlimits) {  // abi.py:196-197
    g_create_kind = EK_BANDLIMIT;
    g_create_msg = "rank must be >= 1";
    return ERR_DOMAIN;
  }
  try {
    std::vector<int> N(bandlimits, bandlimits + rank);
    Plan* p = plan_create(N, node_count, n, m, f1, f2, window, single);
    auto e = std::make_shared<Entry>();
    e->plan = p;
    std::lock_guard<std::mutex> g(g_lock);
    int32_t h = g_next_handle++;
    g_registry[h] = e;
    g_live_buffers += 2;
    return h;
  } catch (const Error& err) {
    g_create_kind = err.kind;
    g_create_msg = err.what();
    return abi_code(err.kind);
  } catch (const std::exception& err) {
    g_create_kind = EK_NFFT;
    g_create_msg = err.what();
    return ERR_INTERNAL;
  }
}

double* alloc_host(int64_t doubles, bool* pinned) {
  size_t bytes = sizeof(double) * (size_t)(doubles > 0 ? doubles : 1);
  void* ptr = nullptr;
  *pinned = false;
  // pinned at every size: copies run at PCIe rate and the host calls can
  // replay their CUDA graph (plan.cu host_call needs pinned buffers)
  if (cudaHostAlloc(&ptr, bytes, cudaHostAllocPortable) == cudaSuccess) {
    *pinned = true;
    memset(ptr, 0, bytes);
    return (double*)ptr;
  }
  cudaGetLastError();
  ptr = calloc(1, bytes);
  if (!ptr) throw std::bad_alloc();
  return (double*)ptr;
}

// Large host copies into the library-owned buffers are split across the host
// cores (the reference's set_fhat / set_f copy too, cabi.py:149-160).
void par_memcpy(void* dst, const void* src, size_t bytes) {
  if (bytes < (1u << 20)) {
    memcpy(dst, src, bytes);
    return;
  }
  const int nt = std::min(16, omp_get_max_threads());
  const size_t chunk = ((bytes + nt - 1) / nt + 63) & ~(size_t)63;
#pragma omp parallel for num_threads(nt) schedule(static, 1)
  for (int t = 0; t < nt; ++t) {
    size_t off = (size_t)t * chunk;
    if (off < bytes) memcpy((char*)dst + off, (const char*)src + off, std::min(chunk, bytes - off));
  }
}

double* fhat_buf(Plan* p) {
  if (!p->fhat_host) p->fhat_host = alloc_host(2 * p->num_freqs, &p->fhat_pinned);
  return p->fhat_host;
}

double* f_buf(Plan* p) {
  if (!p->f_host) p->f_host = alloc_host(2 * p->M, &p->f_pinned);
  return p->f_host;
}

// ABI buffers are complex128; complex64 plans convert at the boundary.
void host_transform(Plan* p, bool forward) {
  double* in = forward ? fhat_buf(p) : f_buf(p);
  double* out = forward ? f_buf(p) : fhat_buf(p);
  int64_t nin = forward ? p->num_freqs : p->M, nout = forward ? p->M : p->num_freqs;
  if (!p->single) {
    if (forward) plan_trafo_host(p, in, out);
    else plan_adjoint_host(p, in, out);
    return;
  }
  std::vector<float> a(2 * nin), b(2 * nout);
  for (int64_t i = 0; i < 2 * nin; ++i) a[i] = (float)in[i];
  if (forward) plan_trafo_host(p, a.data(), b.data());
  else plan_adjoint_host(p, a.data(), b.data());
  for (int64_t i = 0; i < 2 * nout; ++i) out[i] = b[i];
}

}  // namespace

#pragma GCC visibility push(default)
extern "C" {

// ------------------------------------------------------- reference symbols
const char* nfftk_abi_version(void) { return ABI_VERSION; }

int32_t nfftk_create(const int32_t* bandlimits, int32_t rank, int32_t node_count) {
  return do_create(bandlimits, rank, node_count, nullptr, nullptr, nullptr, nullptr, WINDOW_KB, false);
}

int32_t nfftk_create_advanced(const int32_t* bandlimits, int32_t rank, int32_t node_count,
                              const int32_t* fft_lengths, int32_t cutoff, uint32_t flags,
                              uint32_t fft_flags) {
  if (rank >= 1 && !fft_lengths) return ERR_SHAPE;
  // cabi.py:112-124: explicit cutoff (m < 1 -> CutoffError), explicit flag words
  int m = cutoff;
  return do_create(bandlimits, rank, node_count, fft_lengths, &m, &flags, &fft_flags, WINDOW_KB,
                   false);
}

int32_t nfftk_set_x(int32_t h, const double* coords, int64_t len) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  if (len < 0) return ERR_SHAPE;  // abi.py:179-182 (no stored message)
  return guarded(e, [&] {
    plan_set_nodes_host(e->plan, coords, len);
    plan_precompute(e->plan, e->plan->own_stream ? e->plan->own_stream : 0);
  });
}

static int32_t set_complex(int32_t h, const double* values, int64_t len, bool fhat) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  if (len < 0) return ERR_SHAPE;
  return guarded(e, [&] {
    Plan* p = e->plan;
    int64_t count = fhat ? p->num_freqs : p->M;
    if (len != 2 * count)  // cabi.py:149-160
      fail(EK_SHAPE, std::string(fhat ? "fhat" : "f") + " needs " + std::to_string(2 * count) +
                         " interleaved doubles, got " + std::to_string(len));
    double* dst = fhat ? fhat_buf(p) : f_buf(p);
    const size_t bytes = sizeof(double) * 2 * (size_t)count;
    if (!plan_host_upload_begin(p, fhat)) {
      par_memcpy(dst, values, bytes);
      return;
    }
    // chunks: each is copied into the pinned library buffer, then queued for
    // the device -- the PCIe transfer of chunk i runs under the copy of chunk i + 1
    const size_t chunk = (size_t)32 << 20;
    for (size_t off = 0; off < bytes; off += chunk) {
      const size_t nb = std::min(chunk, bytes - off);
      par_memcpy((char*)dst + off, (const char*)values + off, nb);
      plan_host_upload_chunk(p, fhat, off, nb);
    }
    plan_host_upload_end(p, fhat);
  });
}

int32_t nfftk_set_fhat(int32_t h, const double* values, int64_t len) {
  return set_complex(h, values, len, true);
}

int32_t nfftk_set_f(int32_t h, const double* values, int64_t len) {
  return set_complex(h, values, len, false);
}

int32_t nfftk_trafo(int32_t h) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { host_transform(e->plan, true); });
}

int32_t nfftk_adjoint(int32_t h) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { host_transform(e->plan, false); });
}

const double* nfftk_get_f(int32_t h) {
  EntryLock e(h);
  if (!e) return nullptr;
  try { return f_buf(e->plan); } catch (...) { return nullptr; }
}

const double* nfftk_get_fhat(int32_t h) {
  EntryLock e(h);
  if (!e) return nullptr;
  try { return fhat_buf(e->plan); } catch (...) { return nullptr; }
}

int32_t nfftk_last_error(int32_t h) {
  EntryLock e(h);
  return e ? e->err_code : ERR_HANDLE;
}

const char* nfftk_last_error_message(int32_t h) {
  EntryLock e(h);
  if (!e) return "invalid handle";
  return e->err_code ? e->err_msg.c_str() : "";
}

int32_t nfftk_destroy(int32_t h) {
  std::shared_ptr<Entry> e;
  {
    std::lock_guard<std::mutex> g(g_lock);
    auto it = g_registry.find(h);
    if (it == g_registry.end()) return ERR_HANDLE;
    e = it->second;
    g_registry.erase(it);
    g_live_buffers -= 2;
  }
  // waits for a call in flight on this handle; later lookups fail (-1)
  std::lock_guard<std::mutex> g(e->mu);
  delete e->plan;
  e->plan = nullptr;
  return 0;
}

// -------------------------------------------------------------- extensions
const char* nfftk_ext_version(void) { return EXT_VERSION; }

int32_t nfftk_create_ex(const int32_t* bandlimits, int32_t rank, int32_t node_count,
                        const int32_t* fft_lengths, int32_t has_cutoff, int32_t cutoff,
                        int32_t has_flags,
                        uint32_t flags, int32_t has_fft_flags, uint32_t fft_flags,
                        int32_t window, int32_t precision) {
  if (window != WINDOW_KB && window != WINDOW_GAUSS) {
    g_create_kind = EK_NFFT;
    g_create_msg = "unknown window; use 'kaiserbessel' or 'gaussian'";
    return ERR_INTERNAL;
  }
  int m = cutoff;
  return do_create(bandlimits, rank, node_count, fft_lengths, has_cutoff ? &m : nullptr,
                   has_flags ? &flags : nullptr,
                   has_fft_flags ? &fft_flags : nullptr, window, precision == 1);
}

int32_t nfftk_last_create_error_kind(void) { return g_create_kind; }
const char* nfftk_last_create_error_message(void) { return g_create_msg.c_str(); }

int32_t nfftk_last_error_kind(int32_t h) {
  EntryLock e(h);
  return e ? e->err_kind : EK_HANDLE;
}

int32_t nfftk_set_nodes(int32_t h, const double* coords, int64_t len) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_set_nodes_host(e->plan, coords, len); });
}

int32_t nfftk_set_nodes_device(int32_t h, const double* coords, int64_t len, void* stream) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_set_nodes_device(e->plan, coords, len, (cudaStream_t)stream); });
}

int32_t nfftk_precompute(int32_t h) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] {
    Plan* p = e->plan;
    plan_precompute(p, p->own_stream ? p->own_stream : 0);
  });
}

int32_t nfftk_precompute_stream(int32_t h, void* stream) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_precompute(e->plan, (cudaStream_t)stream); });
}

int32_t nfftk_trafo_host(int32_t h, const void* fhat, void* f) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_trafo_host(e->plan, fhat, f); });
}

int32_t nfftk_adjoint_host(int32_t h, const void* f, void* fhat) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_adjoint_host(e->plan, f, fhat); });
}

int32_t nfftk_ndft_host(int32_t h, const double* fhat, double* f) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_ndft_host(e->plan, fhat, f, false); });
}

int32_t nfftk_ndft_adjoint_host(int32_t h, const double* f, double* fhat) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_ndft_host(e->plan, f, fhat, true); });
}

int32_t nfftk_ndft_device(int32_t h, const void* fhat, void* f, void* stream) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_ndft_device(e->plan, fhat, f, false, (cudaStream_t)stream); });
}

int32_t nfftk_ndft_adjoint_device(int32_t h, const void* f, void* fhat, void* stream) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_ndft_device(e->plan, f, fhat, true, (cudaStream_t)stream); });
}

int32_t nfftk_trafo_device(int32_t h, const void* fhat, void* f, void* stream) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_trafo_device(e->plan, fhat, f, (cudaStream_t)stream); });
}

int32_t nfftk_adjoint_device(int32_t h, const void* f, void* fhat, void* stream) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_adjoint_device(e->plan, f, fhat, (cudaStream_t)stream); });
}

int32_t nfftk_spread_device(int32_t h, const void* f, void* stream) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_spread_device(e->plan, f, (cudaStream_t)stream); });
}

int32_t nfftk_interp_device(int32_t h, void* f, void* stream) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_interp_device(e->plan, f, (cudaStream_t)stream); });
}

int32_t nfftk_deconv_cols(int32_t h, int32_t dim, double* out, int64_t len) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] {
    Plan* p = e->plan;
    if (dim < 0 || dim >= p->d) fail(EK_SHAPE, "dimension index outside the plan");
    std::vector<double> c = plan_deconv_cols(p, dim);
    if (len != (int64_t)c.size()) fail(EK_SHAPE, "deconvolution column needs N_i entries");
    memcpy(out, c.data(), sizeof(double) * c.size());
  });
}

int32_t nfftk_adjoint_finish_device(int32_t h, void* fhat, void* stream) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_adjoint_finish_device(e->plan, fhat, (cudaStream_t)stream); });
}

int32_t nfftk_bind_grid(int32_t h, void* dev, int64_t bytes) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_bind_grid(e->plan, dev, bytes); });
}

// params: [d, M, m, window, precision, f1, f2, has_nodes, ready, mode, ntiles, nsubs, width_sum,
//          gridding kernels (0 batch, 1 pipelined row-per-thread, 2 residue-owned), wide nodes]
int32_t nfftk_get_params(int32_t h, int64_t* out, int32_t count) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  Plan* p = e->plan;
  const bool tensor = p->ready && p->mode == MODE_TENSOR && p->d <= MAX_D;
  const int path = !tensor ? 0 : (res_ok(p->geom) ? 2 : (pipe_geometry(p->geom) ? 1 : 0));
  int64_t v[16] = {p->d, p->M, p->m, p->window, p->single ? 1 : 0, (int64_t)p->f1, (int64_t)p->f2,
                   p->has_nodes, p->ready, p->mode, p->ntiles, p->nsubs, (int64_t)p->width_sum,
                   path, p->geom.nwide, p->ready && p->fft3 ? 1 : 0};
  for (int i = 0; i < count && i < 16; ++i) out[i] = v[i];
  return 0;
}

int32_t nfftk_get_sizes(int32_t h, int32_t* N, int32_t* n, int32_t* T, int32_t count) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  Plan* p = e->plan;
  for (int i = 0; i < count && i < p->d; ++i) {
    if (N) N[i] = p->N[i];
    if (n) n[i] = p->n[i];
    if (T) T[i] = i < MAX_D ? p->geom.T[i] : 0;
  }
  return 0;
}

int32_t nfftk_get_window(int32_t h, double* b, double* sigma, int32_t count) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  Plan* p = e->plan;
  for (int i = 0; i < count && i < p->d; ++i) {
    if (b) b[i] = p->b[i];
    if (sigma) sigma[i] = p->sigma[i];
  }
  return 0;
}

int32_t nfftk_phi_hut(int32_t h, int32_t dim, double* out, int64_t len) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] {
    Plan* p = e->plan;
    if (dim < 0 || dim >= p->d) fail(EK_SHAPE, "dimension index outside the plan");
    std::vector<double> t = plan_phi_hut(p, dim);
    if (len != (int64_t)t.size()) fail(EK_SHAPE, "phi_hut needs N_i + 1 entries");
    memcpy(out, t.data(), sizeof(double) * t.size());
  });
}

int32_t nfftk_node_order(int32_t h, int64_t* out, int64_t len) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] {
    if (len != e->plan->M) fail(EK_SHAPE, "node order needs M entries");
    plan_node_order(e->plan, out);
  });
}

int32_t nfftk_psi_tables(int32_t h, double* psi, double* vals, int64_t* idx, int64_t* counts, int64_t len) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] {
    Plan* p = e->plan;
    if (len != p->M * p->d * (2 * p->m + 1)) fail(EK_SHAPE, "psi needs M * d * (2m+1) entries");
    plan_psi_tables(p, psi, vals, idx, counts);
  });
}

int32_t nfftk_lut_tables(int32_t h, double* lut, double* steps, int64_t len) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] {
    if (len != (int64_t)e->plan->d * (LUT_SIZE + 1)) fail(EK_SHAPE, "lut needs d * (2^14 + 1) entries");
    plan_lut_tables(e->plan, lut, steps);
  });
}

int32_t nfftk_window_evals(int32_t h, int64_t* last, int64_t* total) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  if (last) *last = e->plan->window_evals_last;
  if (total) *total = e->plan->window_evals_total;
  return 0;
}

int32_t nfftk_set_psi_policy(int32_t h, int32_t mode) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  if (mode < -1 || mode > MODE_TENSOR) return ERR_DOMAIN;
  e->plan->psi_policy = mode;
  return 0;
}

int32_t nfftk_set_timing(int32_t h, int32_t on) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  e->plan->timing = on != 0;
  return 0;
}

int32_t nfftk_phase_times(int32_t h, double* ms, int64_t* calls, int32_t count, int32_t reset) {
  EntryLock e(h);
  if (!e) return ERR_HANDLE;
  return guarded(e, [&] { plan_phase_times(e->plan, ms, calls, count, reset); });
}

uint64_t nfftk_launch_count(void) { return launch_count(); }

// ---- window math of the library for the host API (window.py:38-181): the
// Python WindowModel evaluates through these, so the closed forms exist once
double nfftk_window_b(int32_t window, int32_t N_i, int32_t n_i, int32_t m) {
  return window_shape(window, N_i, n_i, m);
}

int32_t nfftk_window_values(int32_t window, double n_i, int32_t m, double b_i, const double* t,
                            int64_t count, double* out) {
  if (window != WINDOW_KB && window != WINDOW_GAUSS) return ERR_DOMAIN;
  for (int64_t q = 0; q < count; ++q) out[q] = host_window(window, t[q], n_i, (double)m, b_i);
  return 0;
}

// per entry: 0 ok, 1 KB transform vanishes, 2 not positive (out undefined then)
int32_t nfftk_phi_hat_values(int32_t window, int32_t n_i, int32_t m, double b_i, const int32_t* k,
                             int64_t count, double* out, int32_t* status) {
  if (window != WINDOW_KB && window != WINDOW_GAUSS) return ERR_DOMAIN;
  for (int64_t q = 0; q < count; ++q) status[q] = phi_hat_value(window, k[q], n_i, m, b_i, out + q);
  return 0;
}

double nfftk_bessel_i0(double x) { return host_bessel_i0(x); }

int32_t nfftk_measure_fma_peaks(double* fp64_tflops, double* fp32_tflops) {
  try {
    if (fp64_tflops) *fp64_tflops = measure_fma_tflops(true);
    if (fp32_tflops) *fp32_tflops = measure_fma_tflops(false);
    return 0;
  } catch (...) {
    return ERR_INTERNAL;
  }
}

int32_t nfftk_live_handles(void) {
  std::lock_guard<std::mutex> g(g_lock);
  return (int32_t)g_registry.size();
}

int64_t nfftk_live_buffers(void) {
  std::lock_guard<std::mutex> g(g_lock);
  return g_live_buffers;
}

}  // extern "C"
#pragma GCC visibility pop
