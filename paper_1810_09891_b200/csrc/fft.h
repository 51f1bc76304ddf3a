// Pruned FFT of the oversampled grid for d = 3 (three passes) and d = 2 (two passes) plans (fft.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace nfftk {

// One pass of 1-D line FFTs.  A line is (u, v), v adjacent lines being the
// CTA's group; element e of the line sits at u su + v sv + idx(e) se, where
// idx(e) = e, or the compact band index k + N/2 of slot e when band = N
// (slots outside the band: read as zero / not stored).
struct FftPass {
  int nu, nv;
  int64_t in_su, in_sv, in_se;
  int64_t out_su, out_sv, out_se;
  int in_band, out_band;
  // per group of L / 8 elements (element c L / 8 onwards): compact index of
  // its first element, -1 = outside the band, -2 = edge inside the group
  // (test per element); filled by the launcher
  int in_off[8], out_off[8];
  int scale_in, scale_out;           // x scale col_u[u] col_v[v] col_e[idx] on load / store
  double scale;
  const double* col_e;
  const double* col_u;
  const double* col_v;
  int pad_m;                         // >= 0: store into the ghost-padded grid (u, v = slots of dims 0, 1)
  int pad_d;                         // 3: (u, v, line); 2: (v, line) with pad_n / pad_np at [1], [2]
  int pad_n[3], pad_np[3];
  const void* tw;                    // exp(-2 pi i k / L), k < L, in the pass's precision
};

struct Fft3Geom {
  int d;                             // 3, or 2 (dims at [0], [1])
  int N[3], n[3], np[3];
  int m;
  const double* icol[3];             // device: 1 / (phi_hat_i(k) wscale_i) over k + N_i/2
  double grid_size;
  const void* tw[3];                 // device twiddle tables per dim
};

bool fft3_supported(int d, const int* n, const int* N, bool single);
void fft3_twiddles(int L, bool single, std::vector<unsigned char>& out);
size_t fft3_scratch_elems(const Fft3Geom& q);
// g = F D f_hat: f_hat (N, frequency order) -> the n-grid, dense (row-major)
// or ghost-padded (np, slot s at s + m plus periodic images); scratch holds
// fft3_scratch_elems complex values and must not overlap out
void fft3_forward(bool single, const void* fhat, void* scratch, void* out, bool padded, const Fft3Geom& q,
                  cudaStream_t s);
// f_hat = D^H F^H g: dense n-grid -> f_hat; scratch_a (n0 n1 N2 values) must
// not overlap grid, scratch_b (n0 N1 N2 values) may be the grid itself
void fft3_inverse(bool single, const void* grid, void* scratch_a, void* scratch_b, void* fhat,
                  const Fft3Geom& q, cudaStream_t s);

}  // namespace nfftk
