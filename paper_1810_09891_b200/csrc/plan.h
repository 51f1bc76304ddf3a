// Plan object of the B200 library: parameters (plan.py:124-186), node state
// (plan.py:202-237), device tables (plan.py:249-299) and the transforms
// (transform.py:92-176) issued on a CUDA stream.
#pragma once

#include <cufft.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"
#include "fft.h"
#include "kernels.h"

namespace nfftk {

enum Phase : int {
  PH_DECONV = 0, PH_FFT_FWD, PH_INTERP, PH_ZERO, PH_SPREAD, PH_FFT_INV, PH_PACK,
  PH_H2D, PH_D2H, PH_PAD, PH_FOLD, PH_PERMUTE, PH_COUNT
};

struct Plan {
  // ---- parameters (validated in plan_create)
  int d = 0;
  std::vector<int> N, n;
  int64_t M = 0;
  int m = 0;
  uint32_t f1 = 0, f2 = 0;
  int window = WINDOW_KB;
  bool single = false;              // complex64 grid/arithmetic
  std::vector<double> b, sigma, wscale;
  int64_t num_freqs = 0, grid_size = 0;
  int mode = MODE_DIRECT;           // factor mode chosen at precompute
  int psi_policy = -1;              // -1: follow f1; else force MODE_*

  // ---- state
  bool has_nodes = false, ready = false;
  std::vector<double> x_host;       // host copy of the node set (for x getter / d > 3)
  uint64_t width_sum = 0;
  int64_t window_evals_last = 0, window_evals_total = 0;

  // ---- device resources
  int device = 0;
  cudaStream_t own_stream = nullptr;
  Geom geom{};
  DeconvGeomH dq{};
  int ntiles = 0, nsubs = 0, maxsub = 1024;
  double* x_dev = nullptr;          // (M, d) as given
  double* xs = nullptr;             // (d, M) sorted
  int* perm = nullptr;              // sorted position -> node index
  int* tile_count = nullptr;
  int* tile_start = nullptr;
  int4* subs = nullptr;
  double* psi = nullptr;
  size_t psi_count = 0;
  int4* rec = nullptr;
  unsigned* rrec = nullptr;          // residue-kernel node records (+ one counter of wide nodes at [M + 4])
  void* cublas = nullptr;            // cublasHandle_t for the exact sums (lazy)              // per-node stencil records, sorted order
  double* lut = nullptr;
  double* cols = nullptr;
  void* grid = nullptr;              // dense n-grid (cuFFT, deconvolution)
  bool grid_external = false;
  void* gp = nullptr;                // ghost-padded grid (gridding kernels)
  unsigned* sched = nullptr;         // ticket counters of the persistent spread kernels (SCHED_SLOTS)
  size_t gp_bytes = 0;
  PadGeom pq{};
  alignas(64) unsigned char tmap[128];  // CUtensorMap of gp (halo boxes)
  bool tmap_ready = false;
  void* fhat_dev = nullptr;
  void* f_dev = nullptr;
  // the device copy equals the library-owned host buffer (uploaded by
  // nfftk_set_fhat / nfftk_set_f, or the result of the last host transform):
  // the next host transform skips its host-to-device copy
  bool fhat_dev_cur = false, f_dev_cur = false;
  void* f_sorted = nullptr;         // spread input in tile-sorted order
  cufftHandle fft = 0;
  bool fft_ready = false;
  // pruned three-pass F / F^H with D, D^H and the ghost padding fused in
  // (fft.cu): d = 3 plans on power-of-two grids; cuFFT otherwise
  bool fft3 = false;
  Fft3Geom fq{};
  void* fft_tw[MAX_D] = {nullptr, nullptr, nullptr};

  // ---- host ABI buffers (library-owned, zero-initialised; cabi.py:59-67)
  double* fhat_host = nullptr;
  double* f_host = nullptr;
  bool fhat_pinned = false, f_pinned = false;

  // ---- host-path CUDA graphs (plan_trafo_host / plan_adjoint_host): the
  // H2D copy, the transform's launches and the D2H copy, captured on the
  // second call with the same buffers and plan state, then one
  // cudaGraphLaunch per call.  gen counts the plan-state changes (nodes,
  // tables, grid) that invalidate a captured graph.
  struct HostGraph {
    cudaGraphExec_t exec = nullptr;
    const void* in = nullptr;
    void* out = nullptr;
    uint64_t gen = ~0ull;
    bool skip_h2d = false;
    int seen = 0;
    unsigned long long launches = 0;
  };
  HostGraph hgraph[2];  // 0: trafo, 1: adjoint
  bool graphs_off = false;
  uint64_t gen = 0;

  // ---- instrumentation
  bool timing = false;
  struct Rec { int phase; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> event_pool;
  double phase_ms[PH_COUNT] = {0};
  int64_t phase_calls[PH_COUNT] = {0};

  ~Plan();
  size_t elem_bytes() const { return single ? 8 : 16; }
};

Plan* plan_create(const std::vector<int>& N, int64_t M, const int* n_opt, const int* m_opt,
                  const uint32_t* f1_opt, const uint32_t* f2_opt, int window, bool single);
void plan_set_nodes_host(Plan* p, const double* x, int64_t len);
void plan_set_nodes_device(Plan* p, const double* x_dev, int64_t len, cudaStream_t s);
void plan_precompute(Plan* p, cudaStream_t s);
void plan_trafo_device(Plan* p, const void* fhat, void* f, cudaStream_t s);
void plan_adjoint_device(Plan* p, const void* f, void* fhat, cudaStream_t s);
void plan_spread_device(Plan* p, const void* f, cudaStream_t s);
void plan_interp_device(Plan* p, void* f, cudaStream_t s);
std::vector<double> plan_deconv_cols(const Plan* p, int dim);
void plan_adjoint_finish_device(Plan* p, void* fhat, cudaStream_t s);
// nfftk_set_fhat / nfftk_set_f upload the library buffer while it is being filled
bool plan_host_upload_begin(Plan* p, bool fhat);
void plan_host_upload_chunk(Plan* p, bool fhat, size_t off, size_t bytes);
void plan_host_upload_end(Plan* p, bool fhat);
void plan_trafo_host(Plan* p, const void* fhat, void* f);
void plan_adjoint_host(Plan* p, const void* f, void* fhat);
// exact sums (ndft.cu), complex128 in and out
void plan_ndft_device(Plan* p, const void* in, void* out, bool adjoint, cudaStream_t s);
void plan_ndft_host(Plan* p, const double* in, double* out, bool adjoint);
void plan_node_order(Plan* p, int64_t* out);
void plan_bind_grid(Plan* p, void* dev, int64_t bytes);
void plan_psi_tables(Plan* p, double* psi, double* vals, int64_t* idx, int64_t* counts);
void plan_lut_tables(Plan* p, double* lut, double* steps);
void plan_phase_times(Plan* p, double* ms, int64_t* calls, int nmax, int reset);
std::vector<double> plan_phi_hut(const Plan* p, int dim);
double host_window(int code, double t, double n_i, double m, double b_i);
double host_bessel_i0(double x);
int phi_hat_value(int code, int k, int n_i, int m, double b, double* out);
double window_shape(int code, int N_i, int n_i, int m);

}  // namespace nfftk
