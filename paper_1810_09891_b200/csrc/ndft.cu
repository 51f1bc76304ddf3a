// Exact nonequispaced sums on the device (transform.py:179-234):
//
//   ndft:          f_j   = sum_k fhat_k exp(-2 pi i k.x_j)
//   ndft_adjoint:  fhat_k = sum_j f_j  exp(+2 pi i k.x_j)
//
// O(M |I_N|) work, always complex128 (the reference's exact oracle path).
// The phase factors are separable per dimension, exactly as the reference
// evaluates them (np.exp(sign * 2j * pi * outer(k, x)), k = -N/2 .. N/2-1),
// so the sums split into one dense contraction over the last dimension -- a
// plain ZGEMM (cuBLAS) against a per-chunk phase matrix -- and an elementwise
// reduction over the leading dimensions:
//
//   trafo:   A(j, kr) = sum_kl E_l(j, kl) fhat(kr, kl)            [ZGEMM]
//            f_j      = sum_kr A(j, kr) prod_{i<d-1} E_i(j, k_i)   [k_ndft_reduce]
//   adjoint: B(j, kr) = f_j prod_{i<d-1} E_i(j, k_i)               [k_ndft_spread]
//            fhat(kr, kl) += sum_j E_l(j, kl) B(j, kr)             [ZGEMM]
//
// Nodes are processed in chunks of Mc so the (Mc x prod_{i<d-1} N_i) work
// matrix stays within ~512 MB.  Node order is the caller's (x as given).
#include <cublas_v2.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "plan.h"

namespace nfftk {

namespace {

constexpr double TWO_PI = 6.283185307179586;  // fl(2 * pi) as numpy's 2j * np.pi

// E[jj + k * Mc] = exp(sign 2 pi i kv x_{j0+jj, dim}), kv = k - ceil(Ni / 2)
// (np.arange(-Ni // 2, Ni // 2)); theta = fl(fl(sign 2 pi) * fl(kv * x)) as
// numpy forms (0 + i sign 2 pi) * (kv x).
__global__ void k_phase(const double* __restrict__ x, int d, int dim, int64_t j0, int Mc, int Ni,
                        double sign, double2* __restrict__ E) {
  const int64_t total = (int64_t)Ni * Mc;
  const int k0 = (Ni + 1) / 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(q / Mc), jj = (int)(q - (int64_t)k * Mc);
    const double kx = __dmul_rn((double)(k - k0), x[(j0 + jj) * d + dim]);
    const double th = __dmul_rn(sign * TWO_PI, kx);
    double s, c;
    sincos(th, &s, &c);
    E[q] = make_double2(c, s);
  }
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

struct Lead {
  int nd;                 // number of leading dims (d - 1)
  int N[8];               // their bandwidths
  const double2* E[8];    // their phase tables (N_i x Mc, node fastest)
};

// f_j = sum_kr A(j, kr) prod_i E_i(j, k_i): one thread per node of the chunk,
// kr row-major over the leading dims (coalesced: node index fastest).
__global__ void k_ndft_reduce(const double2* __restrict__ A, Lead L, int Mc, int64_t Nr,
                              double2* __restrict__ f) {
  const int jj = blockIdx.x * blockDim.x + threadIdx.x;
  if (jj >= Mc) return;
  double2 acc = make_double2(0.0, 0.0);
  if (L.nd == 1) {
    for (int k0 = 0; k0 < L.N[0]; ++k0) {
      const double2 t = cmul(A[jj + (int64_t)k0 * Mc], L.E[0][jj + (int64_t)k0 * Mc]);
      acc.x += t.x;
      acc.y += t.y;
    }
  } else if (L.nd == 2) {
    for (int k0 = 0; k0 < L.N[0]; ++k0) {
      double2 s = make_double2(0.0, 0.0);
      const double2* Ar = A + (int64_t)k0 * L.N[1] * Mc;
      for (int k1 = 0; k1 < L.N[1]; ++k1) {
        const double2 t = cmul(Ar[jj + (int64_t)k1 * Mc], L.E[1][jj + (int64_t)k1 * Mc]);
        s.x += t.x;
        s.y += t.y;
      }
      const double2 t = cmul(s, L.E[0][jj + (int64_t)k0 * Mc]);
      acc.x += t.x;
      acc.y += t.y;
    }
  } else {
    for (int64_t kr = 0; kr < Nr; ++kr) {
      int64_t r = kr;
      double2 ph = make_double2(1.0, 0.0);
      for (int i = L.nd - 1; i >= 0; --i) {
        const int ki = (int)(r % L.N[i]);
        r /= L.N[i];
        ph = cmul(ph, L.E[i][jj + (int64_t)ki * Mc]);
      }
      const double2 t = cmul(A[jj + kr * Mc], ph);
      acc.x += t.x;
      acc.y += t.y;
    }
  }
  f[jj] = acc;
}

// B(j, kr) = f_j prod_i E_i(j, k_i)
__global__ void k_ndft_spread(const double2* __restrict__ f, Lead L, int Mc, int64_t Nr,
                              double2* __restrict__ B) {
  const int64_t total = Nr * Mc;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kr = q / Mc;
    const int jj = (int)(q - kr * Mc);
    int64_t r = kr;
    double2 ph = f[jj];
    for (int i = L.nd - 1; i >= 0; --i) {
      const int ki = (int)(r % L.N[i]);
      r /= L.N[i];
      ph = cmul(ph, L.E[i][jj + (int64_t)ki * Mc]);
    }
    B[q] = ph;
  }
}

void cublas_check(cublasStatus_t st, const char* what) {
  if (st != CUBLAS_STATUS_SUCCESS)
    fail(EK_CUDA, std::string("cuBLAS ") + what + " failed (" + std::to_string((int)st) + ")");
}

unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32); }

}  // namespace

void plan_ndft_device(Plan* p, const void* in, void* out, bool adjoint, cudaStream_t s) {
  if (!p->has_nodes) fail(EK_STATE, "plan has no nodes; call set_nodes() first");
  NFFTK_CUDA(cudaSetDevice(p->device >= 0 ? p->device : 0));
  const int d = p->d;
  const int64_t M = p->M;
  // node coordinates on the device (d > 3 keeps them on the host only)
  const double* x = p->x_dev;
  double* x_tmp = nullptr;
  if (!x || d > MAX_D) {
    NFFTK_CUDA(cudaMallocAsync(&x_tmp, sizeof(double) * M * d, s));
    NFFTK_CUDA(cudaMemcpyAsync(x_tmp, p->x_host.data(), sizeof(double) * M * d,
                               cudaMemcpyHostToDevice, s));
    x = x_tmp;
  }
  if (d - 1 > 8) fail(EK_SHAPE, "exact sums support d <= 9");
  const int Nl = p->N[d - 1];
  int64_t Nr = 1;
  for (int i = 0; i + 1 < d; ++i) Nr *= p->N[i];
  const int64_t Mc64 = std::max<int64_t>(1, std::min<int64_t>(M, (int64_t(1) << 25) / std::max<int64_t>(Nr, 1)));
  const int Mc = (int)std::min<int64_t>(Mc64, 1 << 24);
  // workspace: last-dim phases, leading-dim phases, work matrix
  int64_t lead_cols = 0;
  for (int i = 0; i + 1 < d; ++i) lead_cols += p->N[i];
  double2 *El = nullptr, *Elead = nullptr, *W = nullptr;
  NFFTK_CUDA(cudaMallocAsync(&El, sizeof(double2) * (size_t)Nl * Mc, s));
  if (lead_cols) NFFTK_CUDA(cudaMallocAsync(&Elead, sizeof(double2) * (size_t)lead_cols * Mc, s));
  if (d > 1) NFFTK_CUDA(cudaMallocAsync(&W, sizeof(double2) * (size_t)Nr * Mc, s));
  if (!p->cublas) cublas_check(cublasCreate((cublasHandle_t*)&p->cublas), "create");
  cublasHandle_t hb = (cublasHandle_t)p->cublas;
  cublas_check(cublasSetStream(hb, s), "set stream");
  cublas_check(cublasSetMathMode(hb, CUBLAS_DEFAULT_MATH), "math mode");
  const double sign = adjoint ? 1.0 : -1.0;
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  const double2* fin = (const double2*)in;
  double2* fo = (double2*)out;
  for (int64_t j0 = 0; j0 < M; j0 += Mc) {
    const int mc = (int)std::min<int64_t>(Mc, M - j0);
    k_phase<<<grid_for((int64_t)Nl * mc), 256, 0, s>>>(x, d, d - 1, j0, mc, Nl, sign, El);
    count_launch();
    Lead L{};
    L.nd = d - 1;
    int64_t off = 0;
    for (int i = 0; i + 1 < d; ++i) {
      L.N[i] = p->N[i];
      L.E[i] = Elead + off * mc;
      k_phase<<<grid_for((int64_t)p->N[i] * mc), 256, 0, s>>>(x, d, i, j0, mc, p->N[i], sign,
                                                             Elead + off * mc);
      count_launch();
      off += p->N[i];
    }
    if (!adjoint) {
      // A (mc x Nr, col-major, node fastest) = El (mc x Nl) . fhat^T (Nl x Nr)
      double2* A = d > 1 ? W : fo + j0;
      cublas_check(cublasZgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, mc, (int)Nr, Nl, &one,
                               (const cuDoubleComplex*)El, mc, (const cuDoubleComplex*)fin, Nl, &zero,
                               (cuDoubleComplex*)A, mc),
                   "zgemm");
      if (d > 1) {
        k_ndft_reduce<<<(mc + 127) / 128, 128, 0, s>>>(W, L, mc, Nr, fo + j0);
        count_launch();
      }
    } else {
      // fhat^T (Nl x Nr) += El^T (Nl x mc) . B (mc x Nr)
      const double2* B = fin + j0;
      if (d > 1) {
        k_ndft_spread<<<grid_for(Nr * mc), 256, 0, s>>>(fin + j0, L, mc, Nr, W);
        count_launch();
        B = W;
      }
      cublas_check(cublasZgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, Nl, (int)Nr, mc, &one,
                               (const cuDoubleComplex*)El, mc, (const cuDoubleComplex*)B, mc,
                               j0 == 0 ? &zero : &one, (cuDoubleComplex*)fo, Nl),
                   "zgemm");
    }
  }
  NFFTK_CUDA(cudaGetLastError());
  NFFTK_CUDA(cudaFreeAsync(El, s));
  if (Elead) NFFTK_CUDA(cudaFreeAsync(Elead, s));
  if (W) NFFTK_CUDA(cudaFreeAsync(W, s));
  if (x_tmp) NFFTK_CUDA(cudaFreeAsync(x_tmp, s));
}

void plan_ndft_host(Plan* p, const double* in, double* out, bool adjoint) {
  if (!p->has_nodes) fail(EK_STATE, "plan has no nodes; call set_nodes() first");
  NFFTK_CUDA(cudaSetDevice(p->device >= 0 ? p->device : 0));
  cudaStream_t s = nullptr;
  NFFTK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const int64_t nin = adjoint ? p->M : p->num_freqs, nout = adjoint ? p->num_freqs : p->M;
  void *din = nullptr, *dout = nullptr;
  NFFTK_CUDA(cudaMallocAsync(&din, sizeof(double2) * std::max<int64_t>(nin, 1), s));
  NFFTK_CUDA(cudaMallocAsync(&dout, sizeof(double2) * std::max<int64_t>(nout, 1), s));
  NFFTK_CUDA(cudaMemcpyAsync(din, in, sizeof(double2) * nin, cudaMemcpyHostToDevice, s));
  plan_ndft_device(p, din, dout, adjoint, s);
  NFFTK_CUDA(cudaMemcpyAsync(out, dout, sizeof(double2) * nout, cudaMemcpyDeviceToHost, s));
  NFFTK_CUDA(cudaFreeAsync(din, s));
  NFFTK_CUDA(cudaFreeAsync(dout, s));
  NFFTK_CUDA(cudaStreamSynchronize(s));
  NFFTK_CUDA(cudaStreamDestroy(s));
}

}  // namespace nfftk
