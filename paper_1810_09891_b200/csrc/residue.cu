// Residue-owned spread kernel (sm_100a) for d = 3, m = 4, 8^3 tiles:
//   B^H: g[l mod n] += f_j prod_i psi_i(x_ji - l_i / n_i)      kernels.py:209-401
//
// A regular node (stencil 2m = 8 cells wide in every dim) of an 8^3 tile
// touches the halo cells h_i .. h_i + 7, h_i = its cell inside the tile, of
// the 15^3 halo that starts at slot tile * 8 - (m - 1).  Along dim 0 those
// eight cells cover every residue class a mod 8 exactly once, so a CTA of
// 15 x 8 lanes owns the halo rows by (b, a mod 8): lane (b, ra) holds the
// row (a, b, 0..14) with a = ra while the nodes' dim-0 start h_0 is <= ra,
// a = ra + 8 afterwards, as 15 complex register accumulators.
//   * Every lane of a warp whose four b values meet the node's dim-1 window
//     has a row inside the node's dim-0 stencil: 2.75 warps of 4 work per
//     node at 8/11 useful lanes, against 5.8 of 10 at 44% for the
//     row-per-thread kernel (gridding.cu k_spread_pipe, 17^2 rows on 289
//     threads) -- half the per-node instruction stream.
//   * Nodes of a tile arrive sorted by (h_0, h_2, h_1) (k_bin_keys): a lane
//     changes rows once per tile (when h_0 passes ra: the finished row leaves
//     by a TMA bulk fp64 reduction straight away), and the nodes of a run of
//     equal (h_0, h_2) share the unrolled FMA body with static register
//     indices (one switch per run) and the lane's dim-0 factor offset.
//   * One shared-memory row per lane stages the reductions (28.8 KB), so five
//     128-thread CTAs fit an SM; node batches (sten3 PRE_PSI rows, 4-byte
//     records, sorted samples) arrive by TMA bulk copies on an mbarrier ring.
// Nodes with a 2m+1 wide stencil in some dim (n x an exact integer) are
// skipped here and spread by k_wide_nodes (direct window evaluation, atomics).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "async.cuh"
#include "common.cuh"
#include "kernels.h"

namespace nfftk {

struct AresMeta {
  int tile;  // tile of this batch
  int nb;    // nodes (< 0: end of work)
  int last;  // last batch of its subproblem
  int off;   // offset of the records inside the stage (16-byte bulk copies)
};

// Compile-time geometry for cutoff MM on 8^3 tiles: W = 2m residues of dim 0,
// H = W + 7 halo cells per dim, H x W row lanes.
template <typename R, int MM, int NB_, int S_>
struct AresCfg {
  static constexpr int NB = NB_, S = S_;
  static constexpr int W = 2 * MM, H = W + 7, K = 2 * MM + 1;
  static constexpr int ELEM = 2 * (int)sizeof(R);
  static constexpr int FA = 16 / ELEM;                    // samples per 16 bytes
  static constexpr int HO = 8 + K;                        // halo edge of the row-per-thread kernels (rows' index space)
  // PRE_PSI row: sten3 blocks (c128, m <= 4) or halo-indexed [HO | HO | K] (common.cuh pipe_sten3)
  static constexpr bool STEN3 = pipe_sten3(sizeof(R) == 4, MM);
  static constexpr int PR = psi_row_pad<R>(STEN3 ? sten3_count(K) : 2 * HO + K);
  static constexpr int OW0 = STEN3 ? sten3_ow0(K) : 0, OW1 = STEN3 ? sten3_ow1(K) : HO,
                       OWL = STEN3 ? STEN3_OW2 : 2 * HO;
  static constexpr int LANES = H * W;                     // row lanes: b = t / W, ra = t % W
  static constexpr int THREADS = (LANES + 31) / 32 * 32;
  static constexpr int NW = THREADS / 32;
  // staging row: the H cells (complex64: one zero cell in front, so the row
  // starts at an even slot and stays a multiple of 16 bytes -- m and n even),
  // stride a multiple of 16 bytes with an odd number of 16-byte units: eight
  // consecutive rows start in eight different bank groups
  static constexpr int LEAD = ELEM == 8 ? 1 : 0;
  static constexpr int ROW_CELLS = H + LEAD;
  static constexpr int row_stride_bytes() {
    int u = (ROW_CELLS * ELEM + 15) / 16;
    return 16 * (u | 1);
  }
  static constexpr int RS = row_stride_bytes() / ELEM;    // row stride in cells
  static constexpr size_t al(size_t v) { return (v + 15) & ~(size_t)15; }
  static constexpr size_t ROWS_BYTES = al((size_t)THREADS * RS * ELEM);
  static constexpr size_t W_BYTES = al(sizeof(R) * NB * PR);
  static constexpr size_t R_BYTES = al(4 * (size_t)(NB + 4));
  static constexpr size_t F_BYTES = al((size_t)ELEM * (NB + FA));
  static constexpr size_t SB = W_BYTES + R_BYTES + F_BYTES;
  static constexpr size_t RING_OFF = ROWS_BYTES;
  static constexpr size_t CTL_OFF = RING_OFF + S * SB;
  static constexpr size_t SMEM = CTL_OFF + al(16 * (size_t)S + sizeof(AresMeta) * S + 64);
};

// the W last-dim factors of a node (16-byte loads for fp64 rows, 8-byte for fp32 rows)
template <typename R, int W>
__device__ __forceinline__ void load_factors(const R* w, R* o) {
  if constexpr (sizeof(R) == 8) {
    const double2* p = reinterpret_cast<const double2*>(w);
#pragma unroll
    for (int i = 0; i < W / 2; ++i) {
      const double2 v = p[i];
      o[2 * i] = v.x;
      o[2 * i + 1] = v.y;
    }
  } else {
    const float2* p = reinterpret_cast<const float2*>(w);
#pragma unroll
    for (int i = 0; i < W / 2; ++i) {
      const float2 v = p[i];
      o[2 * i] = v.x;
      o[2 * i + 1] = v.y;
    }
  }
}

// One node of a run: the run's nodes are consecutive in the batch (a run is a
// maximal range of consecutive nodes of equal (h_0, h_2) that hit this warp),
// so the factor row, sample and record pointers advance by constants and the
// next node's dim-1 start is read one node ahead.
#define NFFTK_ARES_NODE(H2)                                                                \
  {                                                                                        \
    R s;                                                                                   \
    if constexpr (P::STEN3) s = pw[offa] * pw[P::OW1 + min((unsigned)(b - b0), (unsigned)K)]; \
    else s = pw[offa] * pw[offb];                                                          \
    const unsigned rn = rp[1]; /* next node's record, under this node's FMAs */            \
    const C f = *fp;                                                                       \
    const R cr = f.x * s, ci = f.y * s;                                                    \
    R w2[W];                                                                               \
    load_factors<R, W>(pw + P::OWL, w2);                                                   \
    _Pragma("unroll") for (int t = 0; t < W; ++t) {                                        \
      accr[H2 + t] = fma(cr, w2[t], accr[H2 + t]);                                         \
      acci[H2 + t] = fma(ci, w2[t], acci[H2 + t]);                                         \
    }                                                                                      \
    pw += PR;                                                                              \
    ++fp;                                                                                  \
    ++rp;                                                                                  \
    b0 = (int)((rn >> 3) & 7);                                                             \
  }
#define NFFTK_ARES_CASE(H2)              \
  case H2: {                             \
    const R* pw = ws + j0 * PR;          \
    const C* fp = fv + j0;               \
    const unsigned* rp = rs + j0;        \
    int b0 = (int)((rp[0] >> 3) & 7);    \
    int cnt = __popc(run);               \
    _Pragma("unroll 1") do {             \
      NFFTK_ARES_NODE(H2)                \
    } while (--cnt);                     \
  } break;

template <typename R, int MM, int NB, int S, int BLOCKS, bool GATHER>
__global__ void __launch_bounds__((AresCfg<R, MM, NB, S>::THREADS), BLOCKS)
k_spread_res(cplx_t<R>* __restrict__ grid, const cplx_t<R>* __restrict__ fsorted,
             const cplx_t<R>* __restrict__ funs, const int* __restrict__ perm,
             const R* __restrict__ psi, const unsigned* __restrict__ rrec,
             const int4* __restrict__ subs, int nsubs, Geom g) {
  using C = cplx_t<R>;
  using P = AresCfg<R, MM, NB, S>;
  constexpr int K = P::K, PR = P::PR, W = P::W, H = P::H, NW = P::NW;
  static_assert(NB <= 32, "one ballot per batch");
#ifdef NFFTK_RES_NO_ALT
  constexpr int ALT = 0;
#else
  constexpr int ALT = NW / 2;
#endif
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + P::CTL_OFF);
  unsigned long long* empty = full + S;
  AresMeta* meta = reinterpret_cast<AresMeta*>(empty + S);
  int* pst = reinterpret_cast<int*>(meta + S);  // producer: sub, base, end, tile, pk, next sub, last batch: nodes, slot
  // Sample gather (GATHER): the samples are not read from a
  // sorted copy (k_permute_samples: one more pass over f) but fetched by warp
  // 0 straight from the caller's array, lane l bringing sample
  // funs[perm[base + l]] of the batch with a 16- / 8-byte cp.async whose completion
  // arrives on the batch's mbarrier (32 lane arrivals + the producer's);
  // the lane loads its index one batch ahead.
  constexpr bool gather = GATHER;
  static_assert(!GATHER || NB == 32, "gather: one sample per lane of warp 0");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  C* const myrow = reinterpret_cast<C*>(smem) + (size_t)threadIdx.x * P::RS;  // this lane's staging row
  // pst[5] is the subproblem after pst[0], drawn one ahead so that its node
  // data (PRE_PSI rows, records, samples) is pulled into L2 while the current
  // one is spread: the ring's bulk copies then see L2 latency, not HBM's
  auto load_sub = [&](int s) {
    pst[0] = s;
    if (s < nsubs) {
      const int4 sp = subs[s];
      pst[1] = sp.y;
      pst[2] = sp.y + sp.z;
      pst[3] = sp.x;
      const int nx = next_sub(g, SCHED_SPREAD3, s);
      pst[5] = nx;
      if (nx < nsubs) {
        const int4 sn = subs[nx];
        l2_prefetch(psi + (int64_t)sn.y * PR, (unsigned)(sizeof(R) * PR) * (unsigned)sn.z);
        if (gather) l2_prefetch(perm + (sn.y & ~3), 4u * (unsigned)((sn.z + 6) & ~3));
        else l2_prefetch(fsorted + (sn.y & ~1), (unsigned)sizeof(C) * (unsigned)((sn.z + 2) & ~1));
        l2_prefetch(rrec + (sn.y & ~3), 4u * (unsigned)((sn.z + 6) & ~3));
      }
    }
  };
  auto produce = [&]() {
    const int pk = pst[4];
    const int slot = pk % S;
    if (pk >= S) mbar_wait(empty + slot, ((pk / S) - 1) & 1);
    AresMeta* mt = meta + slot;
    pst[4] = pk + 1;
    if (gather) {
      pst[6] = 0;
      pst[7] = slot;
    }
    if (pst[0] >= nsubs) {
      mt->nb = -1;
      mbar_arrive(full + slot);
      return;
    }
    const int pbase = pst[1], pend = pst[2];
    const int nb = min(NB, pend - pbase);
    const int off = pbase & 3;
    const int rcnt = (nb + off + 3) & ~3;
    constexpr int FA = P::FA;
    const int foff = pbase & (FA - 1);
    mt->tile = pst[3];
    mt->nb = nb;
    mt->last = pbase + nb >= pend;
    mt->off = off;
    unsigned char* st = smem + P::RING_OFF + slot * P::SB;
    const unsigned wb = (unsigned)(sizeof(R) * PR) * nb, rb = 4u * rcnt,
                   fb = gather ? 0u : (unsigned)P::ELEM * ((nb + foff + FA - 1) & ~(FA - 1));
    mbar_expect_tx(full + slot, wb + rb + fb);
    if (gather) pst[6] = nb;
#ifdef NFFTK_NO_STREAM_HINT
    bulk_g2s(st, psi + (int64_t)pbase * PR, wb, full + slot);
    bulk_g2s(st + P::W_BYTES, rrec + (pbase - off), rb, full + slot);
    if (!gather) bulk_g2s(st + P::W_BYTES + P::R_BYTES, fsorted + (pbase - foff), fb, full + slot);
#else
    const unsigned long long pol = l2_evict_first_policy();
    bulk_g2s_stream(st, psi + (int64_t)pbase * PR, wb, full + slot, pol);
    bulk_g2s_stream(st + P::W_BYTES, rrec + (pbase - off), rb, full + slot, pol);
    if (!gather) bulk_g2s_stream(st + P::W_BYTES + P::R_BYTES, fsorted + (pbase - foff), fb, full + slot, pol);
#endif
    if (pbase + nb < pend) pst[1] = pbase + nb;
    else load_sub(pst[5]);
  };
  // warp 0: index of this lane's sample in the batch the producer state points at
  auto fetch_idx = [&]() -> int {
    const int b = pst[1] + lane;
    return pst[0] < nsubs && b < pst[2] ? perm[b] : 0;
  };
  int pidx = 0;
  const unsigned long long gpol = l2_evict_first_policy();
  // warp 0, converged: post the next batch; in gather mode every lane then
  // sends its sample after the batch's byte count is posted
  auto produce_w = [&]() {
    if (gather) __syncwarp();
    if (lane == 0) produce();
    if (gather) {
      __syncwarp();
      const int slot = pst[7];
      if (lane < pst[6])
#ifdef NFFTK_GATHER_NO_HINT
        cp_async_cell<C>(reinterpret_cast<C*>(smem + P::RING_OFF + slot * P::SB + P::W_BYTES + P::R_BYTES) + lane,
                         funs + pidx);
#else
        // read once through a random index: evict-first, so the 1 GiB sample
        // array does not push the prefetched node rows out of L2
        cp_async_cell_hint<C>(reinterpret_cast<C*>(smem + P::RING_OFF + slot * P::SB + P::W_BYTES + P::R_BYTES) + lane,
                              funs + pidx, gpol);
#endif
      cp_async_arrive_noinc(full + slot);
      pidx = fetch_idx();
    }
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full + i, gather ? 33 : 1);
      mbar_init(empty + i, NW);
    }
    pst[4] = 0;
    load_sub((int)blockIdx.x);
  }
  __syncthreads();
  if constexpr (GATHER) {
    if (warp == 0) {
      pidx = fetch_idx();
      for (int i = 0; i < S - 1; ++i) produce_w();
    }
  } else {
    if (threadIdx.x == 0)
      for (int i = 0; i < S - 1; ++i) produce();
  }

  R accr[H], acci[H];
#pragma unroll
  for (int c = 0; c < H; ++c) accr[c] = acci[c] = 0;
  // stage this lane's registers in its shared row and reduce them into the
  // dense grid row (a, b) of the tile (halo cell = slot tile * 8 - (m - 1) + cell)
  auto flush_row = [&](int tile, int a, int b) {
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // the row's previous reduction has read it
    if constexpr (P::LEAD) myrow[0] = C{0, 0};
#pragma unroll
    for (int c = 0; c < H; ++c) {
      C v;
      v.x = accr[c];
      v.y = acci[c];
      myrow[P::LEAD + c] = v;
      accr[c] = acci[c] = 0;
    }
    fence_proxy_async_smem();
    int tc[3];
    tile_of<3>(g, tile, tc);
    int ad = tc[0] * 8 - (MM - 1) + a, bd = tc[1] * 8 - (MM - 1) + b;
    ad += ad < 0 ? g.n[0] : (ad >= g.n[0] ? -g.n[0] : 0);
    bd += bd < 0 ? g.n[1] : (bd >= g.n[1] ? -g.n[1] : 0);
    bulk_red_row_wrapped<R>(grid, ((int64_t)ad * g.n[1] + bd) * g.n[2], tc[2] * 8 - (MM - 1) - P::LEAD, g.n[2],
                            myrow, P::ROW_CELLS);
    asm volatile("cp.async.bulk.commit_group;\n" ::);
  };
  int k = 0;
  for (int par = 0;; par = par ? 0 : ALT) {  // subproblems of this CTA
    // A warp holds 32 / W consecutive b values.  The nodes' dim-1 windows
    // [h_1, h_1 + W - 1] meet the b groups unevenly (m = 4: 50 / 100 / 87.5 /
    // 37.5 % of the nodes) and warp w of every CTA runs on SM sub-partition
    // w mod 4, so a warp takes group w on even subproblems and group
    // w + NW / 2 on odd ones.
    const int t = ((warp + par) % NW) * 32 + lane;
    int b = t / W;
    // keep b in a register of its own: left to itself the compiler may
    // re-derive it from t inside the node loop (a shift + min instead of the
    // fused VIADDMNMX: one more instruction per node visit, C5 spread +0.35 ms)
    if constexpr (sizeof(R) == 8) asm volatile("" : "+r"(b));
    const int ra = t - b * W;
    const bool owner = b < H;
    const int wb_lo = (((warp + par) % NW) * 32) / W, wb_hi = min((((warp + par) % NW) * 32 + 31) / W, H - 1);
    int tile = -1;
    int a = ra;            // this lane's row: the first a = ra (mod W) at or after the nodes' dim-0 start
    bool touched = false;  // a node met this warp's rows since its registers were zeroed
    for (;; ++k) {  // batches of the subproblem
      const int slot = k % S;
      mbar_wait(full + slot, (k / S) & 1);
      const AresMeta mt = meta[slot];
      if (mt.nb < 0) break;
      tile = mt.tile;
      const unsigned char* st = smem + P::RING_OFF + slot * P::SB;
      const R* ws = reinterpret_cast<const R*>(st);
      const unsigned* rs = reinterpret_cast<const unsigned*>(st + P::W_BYTES) + mt.off;
      const C* fv = reinterpret_cast<const C*>(st + P::W_BYTES + P::R_BYTES) +
                    (P::FA > 1 && !gather ? (mt.off & (P::FA - 1)) : 0);
      // Per-batch warp view: lane l holds node l's record; one ballot gives
      // the regular nodes whose dim-1 window meets this warp's b values,
      // another the starts of runs of equal (h_0, h_2).
      const unsigned rl = lane < mt.nb ? rs[lane] : 0u;
      const int bl = (int)((rl >> 3) & 7);
      const bool hit = (rl & RES_REGULAR) && bl <= wb_hi && bl + W - 1 >= wb_lo;
      unsigned mask = __ballot_sync(~0u, hit);
      // runs: consecutive hit nodes of equal (h_0, h_2) (other nodes get a key no run has)
      const unsigned kl = hit ? (rl & 0x1c7u) : 0xffffffffu;
      const unsigned kup = __shfl_up_sync(~0u, kl, 1);
      const unsigned rstart = __ballot_sync(~0u, lane == 0 || kl != kup);
      while (mask) {
        const int j0 = __ffs(mask) - 1;
        const unsigned key = __shfl_sync(~0u, kl, j0);
        const unsigned later = rstart & ~((2u << j0) - 1u);  // run starts after j0 (2u << 31 == 0)
        const unsigned run = later ? mask & ((later & (0u - later)) - 1u) : mask;
        mask &= ~run;
        const int a0 = (int)(key & 7);
        // nodes come by ascending h_0: once it passes a, row a is complete and
        // the lane moves on to the next row of its residue (once per tile for
        // W >= 8)
        if (owner && a < a0) {
          if (touched) flush_row(tile, a, b);
          do a += W;
          while (a < a0);
        }
        touched = true;
        // row a is stencil offset a - h_0 of the run's nodes; halo-indexed
        // PRE_PSI rows hold the factor at the row's cell itself (index + 1:
        // their halo starts one cell earlier)
        const int offa = P::STEN3 ? P::OW0 + (a - a0) : P::OW0 + a + 1;
        // (idle lanes, b >= H, read the block's last entry: zero for regular
        // nodes, so their accumulators stay zero -- they may be row lanes of
        // the next subproblem; sten3 rows clamp onto the block's zero instead)
        const int offb = P::OW1 + min(b + 1, P::HO - 1);
        (void)offb;
        switch (key >> 6) {
          NFFTK_ARES_CASE(0) NFFTK_ARES_CASE(1) NFFTK_ARES_CASE(2) NFFTK_ARES_CASE(3)
          NFFTK_ARES_CASE(4) NFFTK_ARES_CASE(5) NFFTK_ARES_CASE(6) NFFTK_ARES_CASE(7)
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
      if constexpr (GATHER) {
        if (warp == 0) produce_w();
      } else {
        if (threadIdx.x == 0) produce();
      }
      if (mt.last) {
        ++k;
        break;
      }
    }
    if (tile < 0) break;  // end of work
    if (owner && touched) flush_row(tile, a, b);
  }
  if (threadIdx.x == 0) sched_done(g, SCHED_SPREAD3);
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

// ------------------------------------------------ nodes with 2m+1 wide stencils
// One warp per such node (rare: n x an exact integer in some dim): window
// factors evaluated directly (kernels.py:42-53), the stencil walked by the
// lanes, atomics into the dense grid.
template <typename R>
__global__ void __launch_bounds__(256)
k_wide_nodes(cplx_t<R>* __restrict__ grid, const cplx_t<R>* __restrict__ fs, const cplx_t<R>* __restrict__ funs,
             const int* __restrict__ perm, const unsigned* __restrict__ rrec, const double* __restrict__ xs, Geom g) {
  using C = cplx_t<R>;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int K = 2 * g.m + 1;
  for (int64_t base = w0 * 32; base < g.M; base += nw * 32) {
    const int64_t i = base + lane;
    unsigned todo = __ballot_sync(~0u, i < g.M && !(rrec[i] & RES_REGULAR));
    while (todo) {
      const int64_t j = base + __ffs(todo) - 1;
      todo &= todo - 1;
      int64_t lo[3];
      int wd[3];
#pragma unroll
      for (int dim = 0; dim < 3; ++dim) {
        const Stencil st = stencil(xs[dim * g.M + j], g.nd[dim], g.md);
        lo[dim] = st.lo;
        wd[dim] = st.width;
      }
      // lane t < K evaluates the three factors of stencil offset t once
      double fac[3] = {0.0, 0.0, 0.0};
      if (lane < K) {
#pragma unroll
        for (int dim = 0; dim < 3; ++dim)
          if (lane < wd[dim]) fac[dim] = dim_factor(g, dim, xs[dim * g.M + j], lo[dim] + lane) * g.wscale[dim];
      }
      const C fj = perm ? funs[perm[j]] : fs[j];
      const int cells = wd[0] * wd[1] * wd[2];
      for (int q0 = 0; q0 < cells; q0 += 32) {
        const int q = q0 + lane;
        const bool on = q < cells;
        const int qq = on ? q : 0;
        const int t2 = qq % wd[2], t1 = (qq / wd[2]) % wd[1], t0 = qq / (wd[2] * wd[1]);
        const double f0 = __shfl_sync(~0u, fac[0], t0), f1 = __shfl_sync(~0u, fac[1], t1),
                     f2 = __shfl_sync(~0u, fac[2], t2);
        if (!on) continue;
        const double wgt = f0 * f1 * f2;
        const int64_t idx = (floor_mod(lo[0] + t0, g.n[0]) * g.n[1] + floor_mod(lo[1] + t1, g.n[1])) * g.n[2] +
                            floor_mod(lo[2] + t2, g.n[2]);
        atomicAdd(&grid[idx].x, (R)(fj.x * wgt));
        atomicAdd(&grid[idx].y, (R)(fj.y * wgt));
      }
    }
  }
}

// ================================================================ launchers
// d = 3 plans on 8^3 tiles whose halo rows fit one period; complex64 needs m
// and the last grid dim even (16-byte bulk reductions).  The kernel is
// written for any m <= 6 (tests run m = 1..6 with NFFTK_RES_ANY_M), but only
// m = 4 takes it by default: that is where it was measured against the
// row-per-thread kernels and wins (C5: 33.5 -> 20.6 ms c128, 19.3 -> 12.6 ms
// c64); at C3 (m = 6, 64 nodes per tile) it is level or behind (0.341 vs
// 0.325 ms c128, 0.276 vs 0.246 ms c64).
bool res_geometry(const Geom& g, bool single) {
  if (getenv("NFFTK_NO_RES") || getenv("NFFTK_NO_PIPE") || getenv("NFFTK_NO_DENSE_FLUSH")) return false;
  if (g.d != 3 || g.m < 1 || g.m > 6) return false;
  if (g.m != 4 && !getenv("NFFTK_RES_ANY_M")) return false;
  if (single && (g.m % 2 != 0 || g.n[2] % 2 != 0)) return false;
  for (int i = 0; i < 3; ++i)
    if (g.T[i] != 8 || g.n[i] < 8 + 2 * g.m + 1) return false;
  return true;
}

bool res_ok(const Geom& g) {
  return g.res && g.mode == MODE_TENSOR && g.psi && g.rrec && g.psi_pad != 0 && g.dense_flush;
}

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    NFFTK_CUDA(cudaGetDevice(&dev));
    NFFTK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

template <typename R, int MM, int NB, int S, int BLOCKS, bool GATHER>
static void spread_res_gg(void* grid, const void* fs, const void* funs, const int* perm, const int4* subs, int nsubs,
                          const Geom& g, cudaStream_t s) {
  using P = AresCfg<R, MM, NB, S>;
  static_assert(P::SMEM <= 227 * 1024, "residue spread: shared memory");
  if (g.psi_pad != (P::STEN3 ? 2 : 1) || (g.psi_f32 != 0) != (sizeof(R) == 4))
    fail(EK_CUDA, "residue spread: PRE_PSI layout mismatch");
  auto kern = k_spread_res<R, MM, NB, S, BLOCKS, GATHER>;
  NFFTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
  int per_sm = 0;
  NFFTK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, P::THREADS, P::SMEM));
  const int grid_x = std::max(1, std::min(nsubs, sm_count() * std::max(1, per_sm)));
  Geom q = g;
  if ((int64_t)nsubs < 4LL * grid_x) q.sched = nullptr;  // static order (gridding.cu sched_geom)
  kern<<<grid_x, P::THREADS, P::SMEM, s>>>((cplx_t<R>*)grid, (const cplx_t<R>*)fs, (const cplx_t<R>*)funs, perm,
                                          (const R*)g.psi, g.rrec, subs, nsubs, q);
  count_launch();
}

template <typename R, int MM, int NB, int S, int BLOCKS>
static void spread_res_go(void* grid, const void* fs, const void* funs, const int* perm, const int4* subs, int nsubs,
                          const Geom& g, cudaStream_t s) {
  if constexpr (NB == 32) {
    if (perm) {
      spread_res_gg<R, MM, NB, S, BLOCKS, true>(grid, fs, funs, perm, subs, nsubs, g, s);
      return;
    }
  }
  spread_res_gg<R, MM, NB, S, BLOCKS, false>(grid, fs, funs, perm, subs, nsubs, g, s);
}

template <typename R>
static void spread_res_m(void* grid, const void* fs, const void* funs, const int* perm, const int4* subs, int nsubs,
                         const Geom& g, cudaStream_t s) {
  // ring shape / CTAs per SM.  m = 4, c128 (C5): batches of 32 on a 3-deep
  // ring measured best (20.4 ms; <16,3,5> 23.2, <16,4,4> 22.2, <32,2,4> 21.4,
  // <32,4,3> 23.4); NFFTK_RES_VARIANT keeps the others for A/B runs.  The
  // wider rows of m >= 5 take batches of 16.
  const char* e = getenv("NFFTK_RES_VARIANT");
  const int v = e ? atoi(e) : 0;
  switch (g.m) {
    case 1: spread_res_go<R, 1, 32, 3, 4>(grid, fs, funs, perm, subs, nsubs, g, s); break;
    case 2: spread_res_go<R, 2, 32, 3, 4>(grid, fs, funs, perm, subs, nsubs, g, s); break;
    case 3: spread_res_go<R, 3, 32, 3, 3>(grid, fs, funs, perm, subs, nsubs, g, s); break;
    case 4:
      if (v == 1) spread_res_go<R, 4, 16, 3, 5>(grid, fs, funs, perm, subs, nsubs, g, s);
      else if (v == 2) spread_res_go<R, 4, 16, 4, 4>(grid, fs, funs, perm, subs, nsubs, g, s);
      else if (v == 3) spread_res_go<R, 4, 32, 2, 4>(grid, fs, funs, perm, subs, nsubs, g, s);
      else if (v == 4) spread_res_go<R, 4, 32, 4, 3>(grid, fs, funs, perm, subs, nsubs, g, s);
      else spread_res_go<R, 4, 32, 3, 3>(grid, fs, funs, perm, subs, nsubs, g, s);
      break;
    case 5: spread_res_go<R, 5, 16, 3, 2>(grid, fs, funs, perm, subs, nsubs, g, s); break;
    default:
      if (v == 1) spread_res_go<R, 6, 32, 2, 1>(grid, fs, funs, perm, subs, nsubs, g, s);
      else spread_res_go<R, 6, 16, 3, 2>(grid, fs, funs, perm, subs, nsubs, g, s);
      break;
  }
}

// B^H into the dense grid (zeroed by the caller): regular nodes by the
// residue kernel, wide ones (g.nwide of them) by k_wide_nodes.
// the kernel gathers the samples itself (no sorted copy)
bool res_gathers(const Geom& g, bool single) {
  // (the ring shapes with 32-node batches: one sample per lane of warp 0)
  (void)single;
  return res_ok(g) && g.m <= 4 && !getenv("NFFTK_RES_VARIANT") && !getenv("NFFTK_NO_GATHER");
}

void launch_spread_res(bool single, void* grid, const void* fs, const void* funs, const int* perm_all,
                       const double* xs, const int4* subs, int nsubs, const Geom& g, cudaStream_t s) {
  const int* perm = res_gathers(g, single) ? perm_all : nullptr;
  if (single) spread_res_m<float>(grid, fs, funs, perm, subs, nsubs, g, s);
  else spread_res_m<double>(grid, fs, funs, perm, subs, nsubs, g, s);
  if (g.nwide > 0) {
    Geom q = g;
    q.mode = MODE_DIRECT;
    if (single)
      k_wide_nodes<float><<<sm_count() * 4, 256, 0, s>>>((float2*)grid, (const float2*)fs, (const float2*)funs, perm,
                                                         g.rrec, xs, q);
    else
      k_wide_nodes<double><<<sm_count() * 4, 256, 0, s>>>((double2*)grid, (const double2*)fs, (const double2*)funs,
                                                          perm, g.rrec, xs, q);
    count_launch();
  }
}

}  // namespace nfftk
