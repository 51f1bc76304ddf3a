// Shared definitions for the nfftk B200 library: error model, plan geometry,
// device window evaluation.  Reference semantics are cited as
// /root/reference/pkg/src/nfftk/<file>:<line>.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <stdexcept>

namespace nfftk {

// ---------------------------------------------------------------- errors
// Error kinds mirror the reference exception hierarchy (errors.py:4-49);
// abi_code() maps them to the flat ABI codes (cabi.py:39-51, :70-75).
enum ErrKind : int {
  EK_OK = 0,
  EK_BANDLIMIT = 1,        // InvalidBandlimitError
  EK_OVERSAMPLING = 2,     // OversamplingError
  EK_CUTOFF = 3,           // CutoffError
  EK_FLAG = 4,             // InvalidFlagError
  EK_UNSUPPORTED_FLAG = 5, // UnsupportedFlagError (subclass of InvalidFlagError)
  EK_NODE_RANGE = 6,       // NodeRangeError
  EK_SHAPE = 7,            // ShapeError
  EK_STATE = 8,            // PlanStateError
  EK_WINDOW = 9,           // WindowDegenerateError
  EK_NFFT = 10,            // NfftError (base class)
  EK_CUDA = 11,            // device / runtime failure (no reference analogue)
  EK_HANDLE = 12,          // unknown handle (ABI only)
};

constexpr int ERR_HANDLE = -1;
constexpr int ERR_SHAPE = -2;
constexpr int ERR_DOMAIN = -3;
constexpr int ERR_INTERNAL = -9;

inline int abi_code(int kind) {
  switch (kind) {
    case EK_OK: return 0;
    case EK_SHAPE: return ERR_SHAPE;
    case EK_BANDLIMIT: case EK_OVERSAMPLING: case EK_CUTOFF: case EK_FLAG:
    case EK_UNSUPPORTED_FLAG: case EK_NODE_RANGE: case EK_STATE: return ERR_DOMAIN;
    case EK_HANDLE: return ERR_HANDLE;
    default: return ERR_INTERNAL;
  }
}

struct Error : std::runtime_error {
  int kind;
  Error(int k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

[[noreturn]] inline void fail(int kind, const std::string& msg) { throw Error(kind, msg); }

#define NFFTK_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      ::nfftk::fail(::nfftk::EK_CUDA, std::string("CUDA error: ") +                   \
                                          cudaGetErrorString(e_) + " at " #call);    \
  } while (0)

// ------------------------------------------------------------- constants
// f1 flag word, bit values as assigned by the reference (plan.py:31-43).
constexpr uint32_t PRE_PHI_HUT = 1u << 0;
constexpr uint32_t FG_PSI = 1u << 1;
constexpr uint32_t PRE_LIN_PSI = 1u << 2;
constexpr uint32_t PRE_FG_PSI = 1u << 3;
constexpr uint32_t PRE_PSI = 1u << 4;
constexpr uint32_t PRE_FULL_PSI = 1u << 5;
constexpr uint32_t MALLOC_X = 1u << 6;
constexpr uint32_t MALLOC_F_HAT = 1u << 7;
constexpr uint32_t MALLOC_F = 1u << 8;
constexpr uint32_t FFT_OUT_OF_PLACE = 1u << 9;
constexpr uint32_t FFTW_INIT = 1u << 10;
constexpr uint32_t NFFT_SORT_NODES = 1u << 11;
constexpr uint32_t NFFT_OMP_BLOCKWISE_ADJOINT = 1u << 12;
constexpr uint32_t NOOP_F1 = MALLOC_X | MALLOC_F_HAT | MALLOC_F | FFT_OUT_OF_PLACE | FFTW_INIT;
constexpr uint32_t UNSUPPORTED_F1 = FG_PSI | PRE_FG_PSI;
constexpr uint32_t KNOWN_F1 = PRE_PHI_HUT | PRE_LIN_PSI | PRE_PSI | PRE_FULL_PSI |
                              NFFT_SORT_NODES | NFFT_OMP_BLOCKWISE_ADJOINT | NOOP_F1 |
                              UNSUPPORTED_F1;
// f2 (FFTW planner word) is accepted and ignored (plan.py:61-73).
constexpr uint32_t FFTW_DESTROY_INPUT = 1u << 0;
constexpr uint32_t FFTW_ESTIMATE = 1u << 6;
constexpr uint32_t DEFAULT_F2 = FFTW_ESTIMATE | FFTW_DESTROY_INPUT;
constexpr int DEFAULT_CUTOFF = 8;     // plan.py:72
constexpr int LUT_SIZE = 1 << 14;     // plan.py:74

constexpr int WINDOW_KB = 0;          // window.py:32
constexpr int WINDOW_GAUSS = 1;       // window.py:33

// Factor-evaluation modes (kernels.py:25-27); precedence PSI > LUT > DIRECT
// (transform.py:66-82).
constexpr int MODE_DIRECT = 0;
constexpr int MODE_TENSOR = 1;
constexpr int MODE_LUT = 2;

constexpr int MAX_D = 3;              // fast transforms support d <= 3 (transform.py:114)
constexpr int MAX_W = 33;             // 2m+1 for m <= 16

// ------------------------------------------------------------- geometry
// Everything a gridding kernel needs, passed by value.
struct Geom {
  int d;
  int m;
  int code;          // window kind
  int mode;          // MODE_*
  int n[MAX_D];      // oversampled grid
  int T[MAX_D];      // tile edge (cells)
  int H[MAX_D];      // halo edge = T + 2m + 1
  int ntile[MAX_D];  // tiles per dim
  double nd[MAX_D];  // n as double
  double b[MAX_D];   // window shape parameter
  double md;         // m as double
  double wscale[MAX_D];   // window normalisation (1 for c128; 1/phi(0) for c64)
  const double* lut;      // d * (LUT_SIZE+1)  (MODE_LUT)
  double lut_step[MAX_D];
  const double* psi;      // M * psi_row(d, 2m+1) in sorted order (MODE_TENSOR)
  const int4* rec;        // M per-node stencil records, sorted order
  int psi_pad;            // d = 3 pipelined PRE_PSI layout: 0 none (stencil rows), 1 halo-indexed, 2 sten3 blocks
  int pr;                 // PRE_PSI row stride (doubles)
  int64_t M;
  int nt_interp;          // threads per interp CTA
  int np[MAX_D];          // ghost-padded grid (periodic images, halo = one box)
  int HS;                 // halo row stride (elements) of the last dim
  int nb_spread;          // spread node batch size
  int debug;              // NFFTK_DEBUG bits (experiments only; 0 in production)
  int dense_flush;        // pipelined c128 spread reduces into the dense grid (periodic wrap per row), no fold
  int psi_f32;            // PRE_PSI rows stored as fp32 (c64 plans on the pipelined geometries); psi then points at floats
  unsigned* sched;        // plan-owned ticket counters for persistent kernels (SCHED_* slots; null: static order)
  int res;                // residue-owned d = 3 spread (residue.cu): node order and records built for it
  int nwide;              // res: nodes with a 2m+1 wide stencil in some dim (k_wide_nodes)
  const unsigned* rrec;   // res: 4-byte node records, sorted order (RES_* bits)
};

// Residue-owned spread (residue.cu): d = 3, 8^3 tiles.  A regular node
// (stencil 2m wide in every dim) touches halo cells h .. h + 2m - 1, h = its
// cell inside the tile, of the (2m + 7)^3 halo starting at slot
// tile * 8 - (m - 1).
// record: h0 | h1 << 3 | h2 << 6 | regular << 9
constexpr unsigned RES_REGULAR = 1u << 9;

// Dynamic subproblem order for the persistent gridding kernels: CTA b starts at
// subproblem b, then draws tickets gridDim.x + t from a counter, so CTAs that
// drew light tiles take more (clustered nodes: C4).  Each CTA draws exactly
// one failing ticket, so the counter ends at nsubs; the last CTA to finish
// resets it for the next launch on the stream.
enum { SCHED_SPREAD3 = 0, SCHED_SPREAD2 = 2, SCHED_INTERP = 4, SCHED_SLOTS = 8 };
__device__ __forceinline__ int next_sub(const Geom& g, int slot, int cur) {
  if (!g.sched) return cur + (int)gridDim.x;
  return (int)gridDim.x + (int)atomicAdd(g.sched + slot, 1u);
}
__device__ __forceinline__ void sched_done(const Geom& g, int slot) {
  if (!g.sched) return;
  __threadfence();
  if (atomicAdd(g.sched + slot + 1, 1u) == gridDim.x - 1) {
    g.sched[slot] = 0;
    g.sched[slot + 1] = 0;
    __threadfence();
  }
}

// -------------------------------------------------------- device window
// window.py:56-72.  Explicit _rn intrinsics keep the reference's rounding
// sequence (no FMA contraction) so grid-aligned nodes hit u == 0 exactly.
__device__ __forceinline__ double window_kb(double t, double n, double m, double b) {
  double nt = __dmul_rn(n, t);
  double u = __dsub_rn(__dmul_rn(m, m), __dmul_rn(nt, nt));
  if (u > 0.0) {
    double z = sqrt(u);
    return sinh(__dmul_rn(b, z)) / __dmul_rn(3.141592653589793, z);
  }
  if (u < 0.0) {
    double z = sqrt(-u);
    return sin(__dmul_rn(b, z)) / __dmul_rn(3.141592653589793, z);
  }
  return b / 3.141592653589793;
}

__device__ __forceinline__ double window_gauss(double t, double n, double b) {
  double nt = __dmul_rn(n, t);
  return exp(-__dmul_rn(nt, nt) / b) / sqrt(__dmul_rn(3.141592653589793, b));
}

// kernels.py:30-39
__device__ __forceinline__ double lut_factor(const double* row, double step, double t) {
  double u = __dmul_rn(fabs(t), step);
  int64_t idx = (int64_t)u;
  if (idx >= LUT_SIZE) return row[LUT_SIZE];
  double frac = __dsub_rn(u, (double)idx);
  return __dadd_rn(row[idx], __dmul_rn(frac, __dsub_rn(row[idx + 1], row[idx])));
}

// Stencil of node coordinate x along one dim (indexing.py:114-124):
// lo = ceil(n x - m), width = floor(n x + m) - lo + 1; cell = floor(n x).
struct Stencil {
  int64_t lo;
  int width;
  int64_t cell;
};

__device__ __forceinline__ Stencil stencil(double x, double n, double m) {
  double y = __dmul_rn(x, n);
  Stencil s;
  s.lo = (int64_t)ceil(__dsub_rn(y, m));
  s.width = (int)((int64_t)floor(__dadd_rn(y, m)) - s.lo + 1);
  s.cell = (int64_t)floor(y);
  return s;
}

__device__ __forceinline__ int64_t floor_mod(int64_t a, int64_t n) {
  int64_t r = a % n;
  return r < 0 ? r + n : r;
}

// Window factor for node coordinate x at unwrapped cell (kernels.py:47-53).
__device__ __forceinline__ double dim_factor(const Geom& g, int dim, double x, int64_t cell) {
  double off = __dsub_rn(x, (double)cell / g.nd[dim]);
  if (g.mode == MODE_LUT) return lut_factor(g.lut + (size_t)dim * (LUT_SIZE + 1), g.lut_step[dim], off);
  if (g.code == WINDOW_KB) return window_kb(off, g.nd[dim], g.md, g.b[dim]);
  return window_gauss(off, g.nd[dim], g.b[dim]);
}

// PRE_PSI row of one node: d factor vectors of 2m+1, padded to an even count
// so every node row (and, for d = 3, the last-dim vector) is 16-byte aligned
// for bulk copies and 128-bit shared loads.
__host__ __device__ inline int psi_row(int d, int K) { return (d * K + 1) & ~1; }

// Halo-indexed PRE_PSI row (Geom::psi_pad = 1): every leading dim i as a row
// of the tile halo's H_i cells (zero off the stencil, so a halo row reads
// its factor with no stencil test), then the 2m+1 last-dim factors; even
// count.
__host__ __device__ inline int psi_row_halo(int d, const int* H, int K) {
  int s = K;
  for (int i = 0; i + 1 < d; ++i) s += H[i];
  return (s + 1) & ~1;
}

// PRE_PSI row of the d = 3 pipelined kernels (Geom::psi_pad): three blocks of
// K + 1 = 2m + 2 factors -- last dim, dim 0, dim 1 -- each the 2m+1 stencil
// factors of kernels.py:56-72 (zero past the width) plus one zero, so a
// kernel reads dim i's factor for halo cell h of a node whose stencil starts
// at halo cell s as block_i[min((unsigned)(h - s), K)]: off-stencil cells
// land on the zero without a branch.  The last-dim block comes first so its
// factor pairs are 16-byte aligned.  3(K+1) factors per node (m = 4: 240
// bytes) instead of the 2H+K+1 of halo-indexed rows (352 bytes).
// Which layout the d = 3 pipelined kernels use: sten3 for complex128 plans
// with m <= 4 (the run-window spread, C5: 352 -> 240 bytes per node, spread
// and gather time unchanged), halo-indexed rows otherwise -- their spread
// paths index without the stencil-start arithmetic (measured: C3 spread
// 0.319 vs 0.351 ms, C5 c64 spread 20.0 vs 23.1 ms with halo rows).
// Geom::psi_pad = 1 (halo-indexed) or 2 (sten3); NFFTK_HALO_ROWS forces 1.
__host__ __device__ constexpr bool pipe_sten3(bool single, int m) {
#ifdef NFFTK_HALO_ROWS
  return false && single && m;
#else
  return !single && m <= 4;
#endif
}
constexpr int STEN3_OW2 = 0;
__host__ __device__ constexpr int sten3_ow0(int K) { return K + 1; }
__host__ __device__ constexpr int sten3_ow1(int K) { return 2 * (K + 1); }
__host__ __device__ constexpr int sten3_count(int K) { return 3 * (K + 1); }

// PRE_PSI row stride in elements of the factor type: 16-byte rows (fp64
// factors for c128 plans, fp32 factors for c64 plans on the pipelined
// geometries, Geom::psi_f32).
template <typename W>
__host__ __device__ constexpr int psi_row_pad(int count) {
  return sizeof(W) == 8 ? (count + 1) & ~1 : (count + 3) & ~3;
}

template <typename R> struct Cplx;
template <> struct Cplx<double> { using type = double2; };
template <> struct Cplx<float> { using type = float2; };
template <typename R> using cplx_t = typename Cplx<R>::type;

}  // namespace nfftk
