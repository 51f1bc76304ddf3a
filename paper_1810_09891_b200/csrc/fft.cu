// Pruned oversampled FFT for d = 3 and d = 2 plans (sm_100a): F and F^H as
// three (two) passes of hand-written 1-D line FFTs, with D / D^H and the
// ghost-padded layout fused into the first and last pass.
//
//   trafo   g = F (D f_hat)        transform.py:96-104  (deconvolve, zero-pad, fft_nd sign -1)
//   adjoint f_hat = D^H (F^H g)    transform.py:170-176 (fft_nd sign +1, pack, deconvolve)
//
// The reference runs a full n-grid FFT (fft.py:127-139) on a grid of which
// only the N-band (k mod n, |k| < N/2: 1/8 of the cells at sigma = 2) is
// non-zero before F, and only that band is read after F^H.  A line FFT whose
// other coordinates lie outside the band transforms zeros (trafo) or produces
// values nobody reads (adjoint), so the passes run over
//   trafo:   dim 0 on N1 x N2 lines -> dim 1 on n0 x N2 lines -> dim 2 on n0 x n1 lines
//   adjoint: dim 2 on n0 x n1 lines -> dim 1 on n0 x N2 lines -> dim 0 on N1 x N2 lines
// i.e. (1/4 + 1/2 + 1) / 3 = 58% of the butterflies at sigma = 2, and the
// intermediate arrays keep the pruned dims compact (index k + N/2), so the
// passes move 6.2 GB at C5 instead of the 12.9 GB of three full in-place
// passes plus the 6.9 GB of k_deconv_pad, k_pad and k_pack_deconv, whose work
// is done in the first load (x 1/(|I_n| prod phi_hat), zero outside the
// band), the last store of the trafo (every cell written at its ghost-padded
// position and at its periodic images, so the gather's halo is one TMA box)
// and the last store of the adjoint (band only, scaled).
//
// (d = 2: dim 0 on the N1 band columns, then dim 1 on all n0 rows.)
//
// One line = Stockham autosort, radix 8 (then 4), L / 8 threads with 8
// complex registers each, stages exchanged through shared memory; L = 64 ..
// 4096.  Strided
// passes (dims 0, 1) give a CTA G adjacent lines (adjacent last-dim cells):
// lanes run across the lines, so global accesses are 128-byte segments and
// the shared-memory layout [element][line] is conflict-free for any stage.
// The contiguous pass (dim 2) runs lanes along the line over a padded
// [line][element + element / 8] layout.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "fft.h"
#include "kernels.h"

#ifndef NFFTK_FFT_TW_LOADS
#define NFFTK_FFT_TW_LOADS 1
#endif

namespace nfftk {

namespace {

constexpr bool FFT_HALF_GROUP = false;

constexpr int fft_log2(int L) { return L <= 1 ? 0 : 1 + fft_log2(L / 2); }
// radices: as many 8s as possible, the rest 4s (L = 2^p, p >= 6)
constexpr int fft_fours(int L) { return fft_log2(L) % 3 == 0 ? 0 : (fft_log2(L) % 3 == 2 ? 1 : 2); }
constexpr int fft_eights(int L) { return (fft_log2(L) - 2 * fft_fours(L)) / 3; }
constexpr int fft_stages(int L) { return fft_eights(L) + fft_fours(L); }
constexpr int fft_radix(int L, int s) { return s < fft_eights(L) ? 8 : 4; }

template <typename R>
struct Cx {
  using C = cplx_t<R>;
  static __device__ __forceinline__ C add(C a, C b) { return C{a.x + b.x, a.y + b.y}; }
  static __device__ __forceinline__ C sub(C a, C b) { return C{a.x - b.x, a.y - b.y}; }
  static __device__ __forceinline__ C mul(C a, C b) {
    return C{fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x)};
  }
};

// a *= exp(DIR i pi / 4 * Q)
template <typename R, int DIR, int Q>
__device__ __forceinline__ cplx_t<R> rot8(cplx_t<R> a) {
  using C = cplx_t<R>;
  constexpr R h = (R)0.70710678118654752440;
  if constexpr (Q == 2) return DIR < 0 ? C{a.y, -a.x} : C{-a.y, a.x};
  if constexpr (Q == 1) return DIR < 0 ? C{(a.x + a.y) * h, (a.y - a.x) * h} : C{(a.x - a.y) * h, (a.x + a.y) * h};
  if constexpr (Q == 3) return DIR < 0 ? C{(a.y - a.x) * h, -(a.x + a.y) * h} : C{-(a.x + a.y) * h, (a.x - a.y) * h};
  return a;
}

#define NFFTK_FFT2(a, b)        \
  {                             \
    const C t_ = a;             \
    a = Cx<R>::add(t_, b);      \
    b = Cx<R>::sub(t_, b);      \
  }

// radix-4 DFT of (a0, a1, a2, a3); result X0 = a0, X1 = a2, X2 = a1, X3 = a3
template <typename R, int DIR>
__device__ __forceinline__ void fft4(cplx_t<R>& a0, cplx_t<R>& a1, cplx_t<R>& a2, cplx_t<R>& a3) {
  using C = cplx_t<R>;
  NFFTK_FFT2(a0, a2) NFFTK_FFT2(a1, a3)
  a3 = rot8<R, DIR, 2>(a3);
  NFFTK_FFT2(a0, a1) NFFTK_FFT2(a2, a3)
}

// in-register DFT of RAD values, natural order in and out
template <typename R, int DIR, int RAD>
__device__ __forceinline__ void butterfly(cplx_t<R>* v) {
  using C = cplx_t<R>;
  if constexpr (RAD == 4) {
    fft4<R, DIR>(v[0], v[1], v[2], v[3]);
    const C t = v[1];
    v[1] = v[2];
    v[2] = t;
  } else {
    NFFTK_FFT2(v[0], v[4]) NFFTK_FFT2(v[1], v[5]) NFFTK_FFT2(v[2], v[6]) NFFTK_FFT2(v[3], v[7])
    v[5] = rot8<R, DIR, 1>(v[5]);
    v[6] = rot8<R, DIR, 2>(v[6]);
    v[7] = rot8<R, DIR, 3>(v[7]);
    fft4<R, DIR>(v[0], v[1], v[2], v[3]);
    fft4<R, DIR>(v[4], v[5], v[6], v[7]);
    // X0..X7 = a0 a4 a2 a6 a1 a5 a3 a7
    const C x1 = v[4], x3 = v[6], x4 = v[1], x6 = v[3];
    v[1] = x1;
    v[3] = x3;
    v[4] = x4;
    v[6] = x6;
  }
}

// slot e of a length-L line -> compact band index k + N/2, or -1 outside the band (transform.py:39-41)
__device__ __forceinline__ int band_index(int e, int L, int N) {
  const int h = N >> 1;
  return e < h ? e + h : (e >= L - h ? e - L + h : -1);
}

// Lines per CTA.  Strided passes: lanes run across W = 128 / sizeof(complex)
// adjacent lines (8 c128 / 16 c64: 128-byte global segments, one
// shared-memory wavefront per lane group); G = W / 2 halves the CTA (more
// CTAs per SM to overlap the load, butterfly and store phases) and skews the
// element index by e / 8 so that the two elements a wavefront then covers
// fall into different halves of a 128-byte bank row.  Contiguous pass: lanes
// run along the line, G only sets the CTA size.
template <typename R>
struct FftCfg {
  static constexpr int W = 64 / (int)sizeof(R);
#ifndef NFFTK_FFT_GE_DIV
#define NFFTK_FFT_GE_DIV 4
#endif
  static constexpr int GE = W / NFFTK_FFT_GE_DIV;         // contiguous pass: 2 (c128) / 4 (c64) lines per CTA
};

// contiguous pass: one pad element per 128 bytes (c64: per 16 elements when
// the thread count per line allows it, see the kernel's index rules)
template <typename R, int L>
constexpr int fft_pad_shift() {
  return sizeof(R) == 4 && L >= 128 ? 4 : 3;
}

template <typename R, int L, bool EF, int G>
constexpr int fft_smem_elems() {
  return EF ? G * (L + (L >> fft_pad_shift<R, L>())) : (G < FftCfg<R>::W ? (L + (L >> 3)) * G : L * G);
}

constexpr int fft_min_blocks(int threads) { return threads >= 128 ? 1024 / threads : 8; }

// One pass: G lines per CTA, L / 8 threads per line.  Shared-memory index of
// element e of line g: EF: g * pitch + e + (e >> PS) (one pad element per
// 128 bytes); strided: e * G + g, or (e + (e >> 3)) * G + g for the half
// group.  Every access below is base + compile-time offset: reads are at
// e = j + c T, writes at e = d0 + r Ns (Ns >= 8) or 8 j + r, and the pad term
// of such a sum splits into the pad terms of its parts (no carry between
// them).
template <typename R, int L, int DIR, bool EF, int G>
__global__ void __launch_bounds__(G* L / 8, fft_min_blocks(G* L / 8))
k_fft_pass(const cplx_t<R>* __restrict__ in, cplx_t<R>* __restrict__ out, FftPass q) {
  using C = cplx_t<R>;
  constexpr int T = L / 8;
  constexpr int PS = fft_pad_shift<R, L>();
  constexpr bool SKEW = !EF && G < FftCfg<R>::W;
  constexpr int NS = fft_stages(L);
  constexpr bool LAST4 = fft_radix(L, NS - 1) == 4;
  extern __shared__ __align__(16) unsigned char fft_smem[];
  C* buf = reinterpret_cast<C*>(fft_smem);
  const C* __restrict__ tw = reinterpret_cast<const C*>(q.tw);
  const int g = EF ? (int)threadIdx.x / T : (int)threadIdx.x % G;
  const int j = EF ? (int)threadIdx.x % T : (int)threadIdx.x / G;
  const int nvb = q.nv / G;
  const int u = (int)(blockIdx.x / nvb), v = (int)(blockIdx.x % nvb) * G + g;
  // index of element e of this thread's line / offset of an element step c
  auto sidx = [&](int e) -> int {
    return EF ? g * (L + (L >> PS)) + e + (e >> PS) : (SKEW ? (e + (e >> 3)) * G + g : e * G + g);
  };
  auto step = [](int c) -> int { return EF ? c + (c >> PS) : (SKEW ? (c + (c >> 3)) * G : c * G); };

  C x[8];
  // ---- stage 0: radix 8 straight from global memory (zero outside the band)
  {
    const C* src = in + (int64_t)u * q.in_su + (int64_t)v * q.in_sv;
    const int se = (int)q.in_se;
    double fac = 1.0;
    if (q.scale_in) fac = q.scale * (q.col_u ? q.col_u[u] : 1.0) * (q.col_v ? q.col_v[v] : 1.0);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      // band groups: q.in_off[r] is the compact index of element r T (the
      // band edges fall on multiples of T), -1 outside, -2: test per element
      int k = q.in_off[r];
      if (k == -2) k = band_index(j + r * T, L, q.in_band);
      else if (k >= 0) k += j;
      C val = C{0, 0};
      if (k >= 0) {
        val = src[k * se];
        if (q.scale_in) {
          const double f = fac * q.col_e[k];
          val.x = (R)((double)val.x * f);
          val.y = (R)((double)val.y * f);
        }
      }
      x[r] = val;
    }
    butterfly<R, DIR, 8>(x);
    C* w0 = buf + sidx(8 * j);
#pragma unroll
    for (int r = 0; r < 8; ++r) w0[r * (EF ? 1 : G)] = x[r];
  }
  __syncthreads();
  const C* rd = buf + sidx(j);
  // ---- middle and last stages
  int Ns = 8;
#pragma unroll
  for (int s = 1; s < NS; ++s) {
    const int RAD = fft_radix(L, s);
    const bool last = s == NS - 1;
    if (RAD == 8) {
      const int k = j & (Ns - 1);
      const int ts = k * (L / (Ns * 8));
      const C* tp = tw + ts;
      (void)ts;
#pragma unroll
      for (int r = 0; r < 8; ++r) x[r] = rd[step(r * T)];
#if NFFTK_FFT_TW_LOADS == 3
      {
        // three twiddle loads (w, w^2, w^4), the other powers by products:
        // the passes are bound by the load/store unit, not by the FP64 pipe
        C w1 = tp[0], w2 = tp[ts], w4 = tp[3 * ts];
        if (DIR > 0) { w1.y = -w1.y; w2.y = -w2.y; w4.y = -w4.y; }
        const C w3 = Cx<R>::mul(w1, w2), w5 = Cx<R>::mul(w1, w4), w6 = Cx<R>::mul(w2, w4);
        const C w7 = Cx<R>::mul(w3, w4);
        x[1] = Cx<R>::mul(x[1], w1); x[2] = Cx<R>::mul(x[2], w2); x[3] = Cx<R>::mul(x[3], w3);
        x[4] = Cx<R>::mul(x[4], w4); x[5] = Cx<R>::mul(x[5], w5); x[6] = Cx<R>::mul(x[6], w6);
        x[7] = Cx<R>::mul(x[7], w7);
      }
#elif NFFTK_FFT_TW_LOADS == 1
      {
        // one twiddle load, the powers by products (default): the passes are
        // bound by the load/store unit -- C5 F + F^H 3.20 ms with seven loads
        // per stage, 2.65 with three, 2.38 with one; the rounding of the
        // products adds ~1e-16 to the transform's relative error
        C w1 = tp[0];
        if (DIR > 0) w1.y = -w1.y;
        const C w2 = Cx<R>::mul(w1, w1), w3 = Cx<R>::mul(w1, w2), w4 = Cx<R>::mul(w2, w2);
        const C w5 = Cx<R>::mul(w1, w4), w6 = Cx<R>::mul(w2, w4), w7 = Cx<R>::mul(w3, w4);
        x[1] = Cx<R>::mul(x[1], w1); x[2] = Cx<R>::mul(x[2], w2); x[3] = Cx<R>::mul(x[3], w3);
        x[4] = Cx<R>::mul(x[4], w4); x[5] = Cx<R>::mul(x[5], w5); x[6] = Cx<R>::mul(x[6], w6);
        x[7] = Cx<R>::mul(x[7], w7);
      }
#else
#pragma unroll
      for (int r = 1; r < 8; ++r) {
        C w = tp[ts * (r - 1)];
        if (DIR > 0) w.y = -w.y;
        x[r] = Cx<R>::mul(x[r], w);
      }
#endif
      butterfly<R, DIR, 8>(x);
      if (!last) {
        C* wr = buf + sidx((j / Ns) * Ns * 8 + k);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 8; ++r) wr[step(r * Ns)] = x[r];
        __syncthreads();
      }
      // last stage (Ns = T): x[r] is element j + r T
    } else {
      // radix 4: two butterflies per thread, jj = j and j + T; values 4 q + r
#pragma unroll
      for (int qq = 0; qq < 2; ++qq)
#pragma unroll
        for (int r = 0; r < 4; ++r) x[4 * qq + r] = rd[step(qq * T + r * (L / 4))];
      int d0[2];
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        const int jj = j + qq * T;
        const int k = jj & (Ns - 1);
        const int ts = k * (L / (Ns * 4));
        {
          C w1 = tw[ts];  // one load, w^2 and w^3 by products (as in the radix-8 stages)
          if (DIR > 0) w1.y = -w1.y;
          const C w2 = Cx<R>::mul(w1, w1), w3 = Cx<R>::mul(w1, w2);
          x[4 * qq + 1] = Cx<R>::mul(x[4 * qq + 1], w1);
          x[4 * qq + 2] = Cx<R>::mul(x[4 * qq + 2], w2);
          x[4 * qq + 3] = Cx<R>::mul(x[4 * qq + 3], w3);
        }
        butterfly<R, DIR, 4>(x + 4 * qq);
        d0[qq] = (jj / Ns) * Ns * 4 + k;
      }
      if (!last) {
        __syncthreads();
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          C* wr = buf + sidx(d0[qq]);
#pragma unroll
          for (int r = 0; r < 4; ++r) wr[step(r * Ns)] = x[4 * qq + r];
        }
        __syncthreads();
      }
      // last stage (Ns = L / 4): x[4 q + r] is element j + q T + r L / 4
    }
    Ns *= RAD;
  }
  // ---- store: x[i] is element j + EOFF(i)
#define NFFTK_EOFF(i) (LAST4 ? ((i) >> 2) * T + ((i)&3) * (L / 4) : (i)*T)
  if (q.pad_m < 0) {
    C* dst = out + (int64_t)u * q.out_su + (int64_t)v * q.out_sv;
    const int se = (int)q.out_se;
    double fac = 1.0;
    if (q.scale_out) fac = q.scale * (q.col_u ? q.col_u[u] : 1.0) * (q.col_v ? q.col_v[v] : 1.0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int k = q.out_off[NFFTK_EOFF(i) / T];
      if (k == -2) k = band_index(j + NFFTK_EOFF(i), L, q.out_band);
      else if (k >= 0) k += j;
      if (k < 0) continue;
      C val = x[i];
      if (q.scale_out) {
        const double f = fac * q.col_e[k];
        val.x = (R)((double)val.x * f);
        val.y = (R)((double)val.y * f);
      }
      dst[k * se] = val;
    }
  } else {
    // ghost-padded grid: slot s of a dim sits at padded index s + m + k n for
    // every k that lands inside [0, np) (kernels.cu k_pad); u, v are the
    // slots of dims 0 and 1, the line runs along dim 2
    const int m = q.pad_m, np2 = q.pad_np[2];
    auto put_row = [&](C* row) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int pc = j + NFFTK_EOFF(i) + m;
        row[pc] = x[i];
        // images along the line: only its first and last cells have any
        if (NFFTK_EOFF(i) + T + m > L && pc >= L) row[pc - L] = x[i];
        if (NFFTK_EOFF(i) + m + L < np2 && pc + L < np2) row[pc + L] = x[i];
      }
    };
    const bool d3 = q.pad_d == 3, d1 = q.pad_d == 1;
    put_row(d1 ? out : out + ((d3 ? (int64_t)(u + m) * q.pad_np[1] : 0) + (v + m)) * np2);
    // image rows: slots within m (+2) of the edge of dims 0, 1
    const bool ia = d3 && (u + m >= q.pad_n[0] || u + m + q.pad_n[0] < q.pad_np[0]);
    const bool ib = !d1 && (v + m >= q.pad_n[1] || v + m + q.pad_n[1] < q.pad_np[1]);
    if (ia || ib) {
      for (int ka = d3 ? -1 : 0; ka <= (d3 ? 1 : 0); ++ka) {
        const int pa = d3 ? u + m + ka * q.pad_n[0] : 0;
        if (d3 && (pa < 0 || pa >= q.pad_np[0])) continue;
        for (int kb = -1; kb <= 1; ++kb) {
          const int pb = v + m + kb * q.pad_n[1];
          if (pb < 0 || pb >= q.pad_np[1] || (ka == 0 && kb == 0)) continue;
          put_row(out + ((int64_t)pa * q.pad_np[1] + pb) * np2);
        }
      }
    }
  }
#undef NFFTK_EOFF
}

template <typename R, int L, int DIR, bool EF, int G>
void launch_pass_t(const void* in, void* out, const FftPass& q, cudaStream_t s) {
  const size_t smem = sizeof(cplx_t<R>) * fft_smem_elems<R, L, EF, G>();
  NFFTK_CUDA(cudaFuncSetAttribute(k_fft_pass<R, L, DIR, EF, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  const unsigned blocks = (unsigned)((int64_t)q.nu * (q.nv / G));
  k_fft_pass<R, L, DIR, EF, G><<<blocks, G * L / 8, smem, s>>>((const cplx_t<R>*)in, (cplx_t<R>*)out, q);
  count_launch();
}

// lines per CTA of the strided passes: NFFTK_FFT_G=full|half (A/B; default below)
template <typename R>
int strided_group() {
  const char* e = getenv("NFFTK_FFT_G");
  const bool half = e ? e[0] == 'h' : FFT_HALF_GROUP;
  return half ? FftCfg<R>::W / 2 : FftCfg<R>::W;
}

// Long lines (L >= 1024): the CTA holds at most 1024 threads and ~128 KB of
// lines, so the strided groups shrink to 1024 / (L / 8) lines (8 at 1024, 4
// at 2048, 2 at 4096: 128- to 32-byte global segments) on the skewed layout,
// and the contiguous pass takes one or two lines per CTA.
template <typename R, int L>
constexpr int fft_strided_full() {
  return FftCfg<R>::W * (L / 8) <= 1024 ? FftCfg<R>::W : 1024 / (L / 8);
}
template <typename R, int L>
constexpr int fft_contig_group() {
  return FftCfg<R>::GE * (L / 8) <= 512 ? FftCfg<R>::GE : (512 / (L / 8) > 0 ? 512 / (L / 8) : 1);
}

template <typename R, int L, int DIR>
void launch_pass_d(const void* in, void* out, const FftPass& q, bool ef, cudaStream_t s) {
  constexpr int GF = fft_strided_full<R, L>();
  constexpr int GH = GF > 2 ? GF / 2 : GF;
  if (ef && q.nv % fft_contig_group<R, L>() == 0) launch_pass_t<R, L, DIR, true, fft_contig_group<R, L>()>(in, out, q, s);
  else if (ef) launch_pass_t<R, L, DIR, true, 1>(in, out, q, s);
  else if (q.nv % GF == 0 && (GH == GF || strided_group<R>() == FftCfg<R>::W))
    launch_pass_t<R, L, DIR, false, GF>(in, out, q, s);
  else launch_pass_t<R, L, DIR, false, GH>(in, out, q, s);
}

template <typename R, int L>
void launch_pass_l(const void* in, void* out, const FftPass& q, int dir, bool ef, cudaStream_t s) {
  if (dir < 0) launch_pass_d<R, L, -1>(in, out, q, ef, s);
  else launch_pass_d<R, L, 1>(in, out, q, ef, s);
}

static void band_groups(int L, int band, int* off) {
  const int T = L / 8, h = band / 2;
  for (int c = 0; c < 8; ++c) {
    if (!band) off[c] = c * T;
    else if (h % T) off[c] = -2;
    else off[c] = (c + 1) * T <= h ? c * T + h : (c * T >= L - h ? c * T - L + h : -1);
  }
}

template <typename R>
void launch_pass(const void* in, void* out, const FftPass& q0, int L, int dir, bool ef, cudaStream_t s) {
  FftPass q = q0;
  band_groups(L, q.in_band, q.in_off);
  band_groups(L, q.out_band, q.out_off);
  switch (L) {
    case 64: launch_pass_l<R, 64>(in, out, q, dir, ef, s); break;
    case 128: launch_pass_l<R, 128>(in, out, q, dir, ef, s); break;
    case 256: launch_pass_l<R, 256>(in, out, q, dir, ef, s); break;
    case 512: launch_pass_l<R, 512>(in, out, q, dir, ef, s); break;
    case 1024: launch_pass_l<R, 1024>(in, out, q, dir, ef, s); break;
    case 2048: launch_pass_l<R, 2048>(in, out, q, dir, ef, s); break;
    case 4096: launch_pass_l<R, 4096>(in, out, q, dir, ef, s); break;
    default: fail(EK_CUDA, "pruned FFT: unsupported line length " + std::to_string(L));
  }
}

bool len_ok(int L) { return L >= 64 && L <= 4096 && (L & (L - 1)) == 0; }

}  // namespace

// d = 2 or 3, every n_i a supported power of two, N_i even; the band size
// of the last dim (the line coordinate of the strided passes) a multiple of
// the CTA's (half) line group.
bool fft3_supported(int d, const int* n, const int* N, bool single) {
  if (getenv("NFFTK_NO_PRUNED_FFT")) return false;
  if (d < 1 || d > 3) return false;
  const int G = single ? 8 : 4;  // the half group of the strided passes
  for (int i = 0; i < d; ++i)
    if (!len_ok(n[i]) || (N[i] & 1) || N[i] > n[i] || N[i] < 2) return false;
  if (d == 1) return true;  // one contiguous line
  return N[d - 1] % G == 0 && n[d - 2] % G == 0;
}

// exp(-2 pi i k / L), k = 0 .. L-1, rounded from long double
void fft3_twiddles(int L, bool single, std::vector<unsigned char>& out) {
  out.resize((size_t)L * (single ? 8 : 16));
  for (int k = 0; k < L; ++k) {
    // octant symmetry keeps cos / sin exact at the multiples of pi / 2
    const long double a = -2.0L * 3.14159265358979323846264338327950288L * (long double)k / (long double)L;
    long double c = cosl(a), sn = sinl(a);
    if (4 * k == L) { c = 0; sn = -1; }
    if (2 * k == L) { c = -1; sn = 0; }
    if (4 * k == 3 * L) { c = 0; sn = 1; }
    if (single) {
      float* o = reinterpret_cast<float*>(out.data()) + 2 * k;
      o[0] = (float)c;
      o[1] = (float)sn;
    } else {
      double* o = reinterpret_cast<double*>(out.data()) + 2 * k;
      o[0] = (double)c;
      o[1] = (double)sn;
    }
  }
}

size_t fft3_scratch_elems(const Fft3Geom& q) {
  if (q.d == 1) return 0;
  if (q.d == 2) return (size_t)q.n[0] * q.N[1];  // T (n0 x N1)
  // T1 (n0 x N1 x N2) followed by T2 (n0 x n1 x N2)
  return (size_t)q.n[0] * q.N[1] * q.N[2] + (size_t)q.n[0] * q.n[1] * q.N[2];
}

// d = 2: dim 0 on the N1 band columns (deconvolved on load) -> T[a][b'], then
// dim 1 on all n0 rows into the (padded) grid; the adjoint in reverse.
template <typename R>
static void fft2_forward_t(const void* fhat, void* scratch, void* out, bool padded, const Fft3Geom& q,
                           cudaStream_t s) {
  const int64_t N1 = q.N[1], n1 = q.n[1];
  FftPass b{};
  b.nu = 1; b.nv = q.N[1];
  b.in_su = 0; b.in_sv = 1; b.in_se = N1; b.in_band = q.N[0];
  b.out_su = 0; b.out_sv = 1; b.out_se = N1; b.out_band = 0;
  b.scale_in = 1; b.scale = 1.0 / q.grid_size; b.col_e = q.icol[0]; b.col_u = nullptr; b.col_v = q.icol[1];
  b.pad_m = -1; b.tw = q.tw[0];
  launch_pass<R>(fhat, scratch, b, q.n[0], -1, false, s);
  FftPass c{};
  c.nu = 1; c.nv = q.n[0];
  c.in_su = 0; c.in_sv = N1; c.in_se = 1; c.in_band = q.N[1];
  c.out_su = 0; c.out_sv = n1; c.out_se = 1; c.out_band = 0;
  c.pad_m = padded ? q.m : -1; c.pad_d = 2;
  c.pad_n[0] = 1; c.pad_np[0] = 1;
  c.pad_n[1] = q.n[0]; c.pad_np[1] = q.np[0];
  c.pad_n[2] = q.n[1]; c.pad_np[2] = q.np[1];
  c.tw = q.tw[1];
  launch_pass<R>(scratch, out, c, q.n[1], -1, true, s);
}

template <typename R>
static void fft2_inverse_t(const void* grid, void* scratch_a, void* fhat, const Fft3Geom& q, cudaStream_t s) {
  const int64_t N1 = q.N[1], n1 = q.n[1];
  FftPass c{};  // dim 1: rows a of the dense grid -> T[a][b'] (band only)
  c.nu = 1; c.nv = q.n[0];
  c.in_su = 0; c.in_sv = n1; c.in_se = 1; c.in_band = 0;
  c.out_su = 0; c.out_sv = N1; c.out_se = 1; c.out_band = q.N[1];
  c.pad_m = -1; c.tw = q.tw[1];
  launch_pass<R>(grid, scratch_a, c, q.n[1], 1, true, s);
  FftPass b{};  // dim 0: band columns b' -> f_hat[a'][b'], deconvolved on store
  b.nu = 1; b.nv = q.N[1];
  b.in_su = 0; b.in_sv = 1; b.in_se = N1; b.in_band = 0;
  b.out_su = 0; b.out_sv = 1; b.out_se = N1; b.out_band = q.N[0];
  b.scale_out = 1; b.scale = 1.0 / q.grid_size; b.col_e = q.icol[0]; b.col_u = nullptr; b.col_v = q.icol[1];
  b.pad_m = -1; b.tw = q.tw[0];
  launch_pass<R>(scratch_a, fhat, b, q.n[0], 1, false, s);
}

template <typename R>
static void fft3_forward_t(const void* fhat, void* scratch, void* out, bool padded, const Fft3Geom& q,
                           cudaStream_t s) {
  using C = cplx_t<R>;
  const int64_t N1 = q.N[1], N2 = q.N[2], n1 = q.n[1], n2 = q.n[2];
  C* t1 = (C*)scratch;
  C* t2 = t1 + (int64_t)q.n[0] * N1 * N2;
  FftPass a{};  // dim 0: lines (b', c') of f_hat, deconvolved on load -> T1[a][b'][c']
  a.nu = q.N[1]; a.nv = q.N[2];
  a.in_su = N2; a.in_sv = 1; a.in_se = N1 * N2; a.in_band = q.N[0];
  a.out_su = N2; a.out_sv = 1; a.out_se = N1 * N2; a.out_band = 0;
  a.scale_in = 1; a.scale = 1.0 / q.grid_size; a.col_e = q.icol[0]; a.col_u = q.icol[1]; a.col_v = q.icol[2];
  a.pad_m = -1; a.tw = q.tw[0];
  launch_pass<R>(fhat, t1, a, q.n[0], -1, false, s);
  FftPass b{};  // dim 1: lines (a, c') of T1 -> T2[a][b][c']
  b.nu = q.n[0]; b.nv = q.N[2];
  b.in_su = N1 * N2; b.in_sv = 1; b.in_se = N2; b.in_band = q.N[1];
  b.out_su = n1 * N2; b.out_sv = 1; b.out_se = N2; b.out_band = 0;
  b.pad_m = -1; b.tw = q.tw[1];
  launch_pass<R>(t1, t2, b, q.n[1], -1, false, s);
  FftPass c{};  // dim 2: lines (a, b) of T2 -> the n-grid (dense or ghost-padded)
  c.nu = q.n[0]; c.nv = q.n[1];
  c.in_su = n1 * N2; c.in_sv = N2; c.in_se = 1; c.in_band = q.N[2];
  c.out_su = n1 * n2; c.out_sv = n2; c.out_se = 1; c.out_band = 0;
  c.pad_m = padded ? q.m : -1; c.pad_d = 3;
  for (int i = 0; i < 3; ++i) { c.pad_n[i] = q.n[i]; c.pad_np[i] = q.np[i]; }
  c.tw = q.tw[2];
  launch_pass<R>(t2, out, c, q.n[2], -1, true, s);
}

template <typename R>
static void fft3_inverse_t(const void* grid, void* scratch_a, void* scratch_b, void* fhat, const Fft3Geom& q,
                           cudaStream_t s) {
  using C = cplx_t<R>;
  const int64_t N1 = q.N[1], N2 = q.N[2], n1 = q.n[1], n2 = q.n[2];
  C* t2 = (C*)scratch_a;  // n0 x n1 x N2
  C* t1 = (C*)scratch_b;  // n0 x N1 x N2
  FftPass c{};  // dim 2: lines (a, b) of the dense grid -> T2[a][b][c'] (band only)
  c.nu = q.n[0]; c.nv = q.n[1];
  c.in_su = n1 * n2; c.in_sv = n2; c.in_se = 1; c.in_band = 0;
  c.out_su = n1 * N2; c.out_sv = N2; c.out_se = 1; c.out_band = q.N[2];
  c.pad_m = -1; c.tw = q.tw[2];
  launch_pass<R>(grid, t2, c, q.n[2], 1, true, s);
  FftPass b{};  // dim 1: lines (a, c') -> T1[a][b'][c']
  b.nu = q.n[0]; b.nv = q.N[2];
  b.in_su = n1 * N2; b.in_sv = 1; b.in_se = N2; b.in_band = 0;
  b.out_su = N1 * N2; b.out_sv = 1; b.out_se = N2; b.out_band = q.N[1];
  b.pad_m = -1; b.tw = q.tw[1];
  launch_pass<R>(t2, t1, b, q.n[1], 1, false, s);
  FftPass a{};  // dim 0: lines (b', c') -> f_hat[a'][b'][c'], deconvolved on store
  a.nu = q.N[1]; a.nv = q.N[2];
  a.in_su = N2; a.in_sv = 1; a.in_se = N1 * N2; a.in_band = 0;
  a.out_su = N2; a.out_sv = 1; a.out_se = N1 * N2; a.out_band = q.N[0];
  a.scale_out = 1; a.scale = 1.0 / q.grid_size; a.col_e = q.icol[0]; a.col_u = q.icol[1]; a.col_v = q.icol[2];
  a.pad_m = -1; a.tw = q.tw[0];
  launch_pass<R>(t1, fhat, a, q.n[0], 1, false, s);
}

// d = 1: the one line, f_hat -> (padded) grid and back
template <typename R>
static void fft1_t(const void* in, void* out, bool forward, bool padded, const Fft3Geom& q, cudaStream_t s) {
  FftPass c{};
  c.nu = 1; c.nv = 1;
  c.in_se = 1; c.out_se = 1;
  c.in_band = forward ? q.N[0] : 0;
  c.out_band = forward ? 0 : q.N[0];
  c.scale_in = forward; c.scale_out = !forward;
  c.scale = 1.0 / q.grid_size; c.col_e = q.icol[0]; c.col_u = nullptr; c.col_v = nullptr;
  c.pad_m = forward && padded ? q.m : -1; c.pad_d = 1;
  for (int i = 0; i < 3; ++i) { c.pad_n[i] = 1; c.pad_np[i] = 1; }
  c.pad_n[2] = q.n[0]; c.pad_np[2] = q.np[0];
  c.tw = q.tw[0];
  launch_pass<R>(in, out, c, q.n[0], forward ? -1 : 1, true, s);
}

void fft3_forward(bool single, const void* fhat, void* scratch, void* out, bool padded, const Fft3Geom& q,
                  cudaStream_t s) {
  if (q.d == 1) {
    if (single) fft1_t<float>(fhat, out, true, padded, q, s);
    else fft1_t<double>(fhat, out, true, padded, q, s);
    return;
  }
  if (q.d == 2) {
    if (single) fft2_forward_t<float>(fhat, scratch, out, padded, q, s);
    else fft2_forward_t<double>(fhat, scratch, out, padded, q, s);
    return;
  }
  if (single) fft3_forward_t<float>(fhat, scratch, out, padded, q, s);
  else fft3_forward_t<double>(fhat, scratch, out, padded, q, s);
}

void fft3_inverse(bool single, const void* grid, void* scratch_a, void* scratch_b, void* fhat,
                  const Fft3Geom& q, cudaStream_t s) {
  if (q.d == 1) {
    if (single) fft1_t<float>(grid, fhat, false, false, q, s);
    else fft1_t<double>(grid, fhat, false, false, q, s);
    return;
  }
  if (q.d == 2) {
    if (single) fft2_inverse_t<float>(grid, scratch_a, fhat, q, s);
    else fft2_inverse_t<double>(grid, scratch_a, fhat, q, s);
    return;
  }
  if (single) fft3_inverse_t<float>(grid, scratch_a, scratch_b, fhat, q, s);
  else fft3_inverse_t<double>(grid, scratch_a, scratch_b, fhat, q, s);
}

}  // namespace nfftk
