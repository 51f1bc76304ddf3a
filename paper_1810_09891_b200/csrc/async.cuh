// Async-copy / mbarrier / TMA PTX wrappers shared by the gridding kernels
// (gridding.cu, fold.cu).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace nfftk {

__device__ __forceinline__ size_t a16(size_t v) { return (v + 15) & ~(size_t)15; }

template <int D>
__device__ __forceinline__ void tile_of(const Geom& g, int tile, int* tc) {
  int t = tile;
#pragma unroll
  for (int i = D - 1; i >= 0; --i) {
    tc[i] = t % g.ntile[i];
    t /= g.ntile[i];
  }
}

// ------------------------------------------------------- async copy PTX
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
// the executing thread's earlier cp.async copies arrive on bar when they
// land; .noinc: the arrival is part of the barrier's expected count
__device__ __forceinline__ void cp_async_arrive_noinc(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// cp.async of one cell with an L2 cache policy (createpolicy, e.g. evict-first
// for data read once through a random index)
template <typename C>
__device__ __forceinline__ void cp_async_cell_hint(C* sdst, const C* gsrc, unsigned long long pol) {
  if constexpr (sizeof(C) == 16)
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
                 "l"(pol));
  else
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
                 "l"(pol));
}

template <typename C>
__device__ __forceinline__ void cp_async_cell(C* sdst, const C* gsrc) {
  if constexpr (sizeof(C) == 16) cp_async16(sdst, gsrc);
  else cp_async8(sdst, gsrc);
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
#ifdef NFFTK_MBAR_HINT
  // A/B: let a failed try_wait suspend the warp for up to the hinted time
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"((unsigned)NFFTK_MBAR_HINT)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// TMA: L2 prefetch of a halo box (no shared-memory destination)
__device__ __forceinline__ void tma_prefetch_box3(const CUtensorMap* tm, const int* c) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(tm),
               "r"(c[0]), "r"(c[1]), "r"(c[2])
               : "memory");
}

// L2 prefetch of a contiguous global range (16-byte aligned address, size a multiple of 16)
__device__ __forceinline__ void l2_prefetch(const void* gsrc, unsigned bytes) {
  if (bytes)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(gsrc), "r"(bytes) : "memory");
}

// TMA: whole halo box of the padded grid -> shared memory
template <int D>
__device__ __forceinline__ void tma_load_box(void* sdst, const CUtensorMap* tm, const int* c,
                                             unsigned long long* bar) {
  if constexpr (D == 3) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(sdst)),
        "l"(tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(smem_u32(bar))
        : "memory");
  } else if constexpr (D == 2) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(sdst)),
        "l"(tm), "r"(c[0]), "r"(c[1]), "r"(smem_u32(bar))
        : "memory");
  }
}

__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The same copy for streamed-once data (node batches): L2 evict-first, so the
// stream does not push the grid lines the tiles share out of L2.
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_stream(void* sdst, const void* gsrc, unsigned bytes,
                                                unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// TMA bulk reduction shared -> global (L2 performs the adds)
template <typename R>
__device__ __forceinline__ void bulk_red_add(void* gdst, const void* ssrc, unsigned bytes) {
  if constexpr (sizeof(R) == 8)
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
  else
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;\n" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
// One staged halo row into the DENSE grid: cells [c0, c0 + len) of the row
// starting at dense index rowbase, c0 in [-n2, n2), wrapped periodically
// (kernels.py:47 slot arithmetic) -- at most two bulk reductions.  Both
// pieces stay 16-byte aligned: c128 cells are 16 bytes; c64 needs c0, len
// and n2 even (spread_dense_ok).
template <typename R>
__device__ __forceinline__ void bulk_red_row_wrapped(cplx_t<R>* grid, int64_t rowbase, int c0, int n2,
                                                     const cplx_t<R>* src, int len) {
  const int c = c0 < 0 ? c0 + n2 : c0;
  const int first = min(len, n2 - c);
  bulk_red_add<R>(grid + rowbase + c, src, (unsigned)(first * sizeof(cplx_t<R>)));
  if (first < len)
    bulk_red_add<R>(grid + rowbase, src + first, (unsigned)((len - first) * sizeof(cplx_t<R>)));
}

__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\n" ::);
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

}  // namespace nfftk
