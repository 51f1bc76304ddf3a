// Host-side launchers for the kernels in kernels.cu.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"

namespace nfftk {

struct PadGeom {
  int d;
  int n[MAX_D];
  int np[MAX_D];
  int m;
};

struct DeconvGeomH {
  int d;
  int N[MAX_D];
  int n[MAX_D];
  const double* icol[MAX_D];  // device: 1 / (phi_hat_i(k) * wscale_i) for k + N_i/2
  double grid_size;
};

unsigned long long launch_count();
void count_launch();
void add_launches(unsigned long long n);
int spread_threads(const Geom& g);

void launch_check_range(const double* x, int64_t count, unsigned long long* first_bad,
                        cudaStream_t s);
void bin_and_sort(const double* x_dev, int64_t M, const Geom& g, int maxsub, int ntiles,
                  int* perm, double* xs, int* tile_count, int* tile_start, int4** subs,
                  int* nsubs, cudaStream_t s);
unsigned long long sum_widths(const double* xs, int64_t M, const Geom& g, cudaStream_t s);
void build_psi(const double* xs, int64_t M, const Geom& g, void* psi, cudaStream_t s);
bool pipe_geometry(const Geom& g);
bool spread_dense_ok(const Geom& g, int elem_bytes);
void build_recs(const double* xs, int64_t M, const Geom& g, int4* rec, unsigned* rrec, unsigned* nwide,
                cudaStream_t s);
// residue-owned d = 3 spread (residue.cu)
bool res_geometry(const Geom& g, bool single);
bool res_ok(const Geom& g);
bool res_gathers(const Geom& g, bool single);
bool spread_gathers(const Geom& g, bool single);
void launch_spread_res(bool single, void* grid, const void* fs, const void* f, const int* perm, const double* xs,
                       const int4* subs, int nsubs, const Geom& g, cudaStream_t s);

void lex_order(const double* x_dev, int64_t M, const Geom& g, int* order, cudaStream_t s);
void psi_reference(const double* x_dev, int64_t M, const Geom& g, double* psi, double* vals, int64_t* idx,
                   int64_t* counts, cudaStream_t s);

void launch_deconv(bool single, const void* fhat, void* grid, const DeconvGeomH& q, cudaStream_t s);
void launch_pack(bool single, const void* grid, void* fhat, const DeconvGeomH& q, cudaStream_t s);
void launch_interp(bool single, const void* tmap, const void* gp, void* f, const double* xs,
                   const int* perm, const int4* subs, int nsubs, const Geom& g, cudaStream_t s);
void launch_permute(bool single, const void* f, const int* perm, int64_t M, void* fs, cudaStream_t s);
void launch_pad(bool single, const void* g0, void* gp, const PadGeom& q, cudaStream_t s);
void launch_fold(bool single, const void* gp, void* g0, const PadGeom& q, cudaStream_t s);
size_t spread_smem_nb(const Geom& g, int elem_bytes, int nb);
void launch_spread(bool single, void* grid, const void* f, void* fs, const double* xs,
                   const int* perm, const int4* subs, int nsubs, const Geom& g, cudaStream_t s);

double measure_fma_tflops(bool fp64);

size_t interp_smem(const Geom& g, int elem_bytes, int threads);
size_t spread_smem(const Geom& g, int elem_bytes);

}  // namespace nfftk
