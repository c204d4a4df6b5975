// bn_common.cuh — device building blocks shared by the three hot-path kernels.
//
//   * 128-bit global/shared vector moves,
//   * the carry-propagation scan of §2: per-thread
//     sequential fold over L limbs ("efficient sequentialization",
//     PAPER.md:283-292), a warp-level scan done with two ballots and one
//     integer add, and a CTA-level scan of warp aggregates through shared
//     memory (the hierarchical thread/warp/block decomposition of
//     PAPER.md:289-292).
//
// The scan computes the same exclusive scan as the paper's carry_op_eff
// (Fig. 3) over the (ov, mx) = (generate, propagate) pairs
// of each limb: for a chunk, g = carry out with carry-in 0 and p = "every
// limb sum is 0xFFFFFFFF"; carry-out(cin) = g | (p & cin).  Over the lanes of
// a warp with G = ballot(g), P = ballot(p), X = G|P, the carry into lane i is
// bit i of (X + G + c0) ^ X ^ G: integer addition IS the carry-lookahead
// network (tests/test_scan_model.py pins this against the sequential fold on
// all 3^8 8-lane patterns).  Instances never exchange carries: the top lane of
// each segment has its (g, p) cleared (reading R1: each instance's
// carry-in is 0 and its top carry-out is dropped).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "bn_config.h"

#define BN_DEV __device__ __forceinline__

namespace bn {

// ---------------------------------------------------------------- vector I/O
BN_DEV uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
BN_DEV void stg_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

template <int L>
BN_DEV void load_limbs(uint32_t (&r)[L], const uint32_t* src) {
  static_assert(L % 4 == 0, "L must be a multiple of 4");
#pragma unroll
  for (int v = 0; v < L / 4; v++) {
    uint4 x = ldg_stream(reinterpret_cast<const uint4*>(src) + v);
    r[4 * v + 0] = x.x; r[4 * v + 1] = x.y; r[4 * v + 2] = x.z; r[4 * v + 3] = x.w;
  }
}
template <int L>
BN_DEV void store_limbs(uint32_t* dst, const uint32_t (&r)[L]) {
#pragma unroll
  for (int v = 0; v < L / 4; v++)
    stg_stream(reinterpret_cast<uint4*>(dst) + v,
               make_uint4(r[4 * v + 0], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]));
}
// Coherent (L2) 128-bit load / write-back store, for buffers that the same
// kernel writes and later reads back (the fused workloads' per-CTA workspace:
// ld.global.nc must not be used on data written during the kernel).
template <int L>
BN_DEV void ldcg_limbs(uint32_t (&r)[L], const uint32_t* src) {
#pragma unroll
  for (int v = 0; v < L / 4; v++) {
    uint4 x = __ldcg(reinterpret_cast<const uint4*>(src) + v);
    r[4 * v + 0] = x.x; r[4 * v + 1] = x.y; r[4 * v + 2] = x.z; r[4 * v + 3] = x.w;
  }
}
template <int L>
BN_DEV void stg_limbs(uint32_t* dst, const uint32_t (&r)[L]) {
#pragma unroll
  for (int v = 0; v < L / 4; v++)
    reinterpret_cast<uint4*>(dst)[v] = make_uint4(r[4 * v + 0], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
}
// HBM operand (ld.global.nc, streaming) or in-kernel workspace (ld.global.cg)
template <bool WS, int L>
BN_DEV void load_any(uint32_t (&r)[L], const uint32_t* src) {
  if constexpr (WS) ldcg_limbs<L>(r, src);
  else load_limbs<L>(r, src);
}
template <bool WS, int L>
BN_DEV void store_any(uint32_t* dst, const uint32_t (&r)[L]) {
  if constexpr (WS) stg_limbs<L>(dst, r);
  else store_limbs<L>(dst, r);
}

template <int L>
BN_DEV void lds_limbs(uint32_t (&r)[L], const uint32_t* src) {
#pragma unroll
  for (int v = 0; v < L / 4; v++) {
    uint4 x = reinterpret_cast<const uint4*>(src)[v];
    r[4 * v + 0] = x.x; r[4 * v + 1] = x.y; r[4 * v + 2] = x.z; r[4 * v + 3] = x.w;
  }
}
template <int L>
BN_DEV void sts_limbs(uint32_t* dst, const uint32_t (&r)[L]) {
#pragma unroll
  for (int v = 0; v < L / 4; v++)
    reinterpret_cast<uint4*>(dst)[v] = make_uint4(r[4 * v + 0], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
}

// Shared-memory swizzle for arrays accessed as Q consecutive words per
// thread with 128-bit accesses (Q = 8 or 16) and also, in some kernels, in a
// pass layout (consecutive threads -> consecutive words): XOR the 16-byte
// chunk index inside each 32-word row with the row number's low bits.  A
// permutation inside every aligned 16-word group; the 8 threads of a
// quarter-warp then hit 8 distinct 16-byte bank groups instead of Q/4-way
// conflicts (tests/test_ntt_layout.py::test_epilogue_swizzle_conflict_free).
// S = false: plain row-major (kernels whose issue slots are the binding limit
// measured faster without the extra address arithmetic).
template <int Q, bool S = true>
BN_DEV int cswz(int k) {
  static_assert(Q == 8 || Q == 16, "Q words per thread");
  if constexpr (S) return k ^ (((k >> 5) & (Q / 4 - 1)) << 2);
  else return k;
}

// cp.async (LDGSTS) 16-byte global -> shared copy; !valid zero-fills the
// destination without reading the source.
BN_DEV void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gsrc), "r"(sz) : "memory");
}
BN_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
BN_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ------------------------------------------------------------- mbarrier / TMA
// Completion barriers for bulk (TMA) copies into shared memory.
BN_DEV uint32_t mbar_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
BN_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar_addr(bar)), "r"(count) : "memory");
}
BN_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar_addr(bar)), "r"(bytes)
               : "memory");
}
BN_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(mbar_addr(bar)),
      "r"(parity)
      : "memory");
}
BN_DEV void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          mbar_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(mbar_addr(bar))
      : "memory");
}
// ------------------------------------------------------------- carry scan

// Mask with bit l set for every lane l that is the top lane of a TPI-lane
// segment (TPI a power of two <= 32).
template <int TPI>
constexpr uint32_t seg_top_mask() {
  uint32_t m = 0;
  for (int l = TPI - 1; l < 32; l += TPI) m |= 1u << l;
  return m;
}

// Thread-level map + fold (PAPER.md:150-157 step (1), carry_op over the
// thread's L limbs), done with the hardware carry chain: s = x + y as one
// 32L-bit sum (intra-chunk carries included), g = its carry-out (the fold's
// generate with carry-in 0), p = "s is all ones" (the fold's propagate: a
// carry-in would ripple through every limb).  Groups of 4 limbs per asm
// block; the carry between groups travels in a register.
BN_DEV uint32_t add4_cc(uint32_t (&s)[4], const uint32_t* x, const uint32_t* y, uint32_t cin) {
  uint32_t c;
  asm("add.cc.u32 %0, %5, 0xFFFFFFFF;\n\t"  // CC.carry = (cin != 0), cin in {0, 1}
      "addc.cc.u32 %0, %6, %10;\n\t"
      "addc.cc.u32 %1, %7, %11;\n\t"
      "addc.cc.u32 %2, %8, %12;\n\t"
      "addc.cc.u32 %3, %9, %13;\n\t"
      "addc.u32 %4, 0, 0;"
      : "=&r"(s[0]), "=&r"(s[1]), "=&r"(s[2]), "=&r"(s[3]), "=r"(c)
      : "r"(cin), "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]));
  return c;
}
BN_DEV uint32_t inc4_cc(uint32_t (&s)[4], uint32_t cin) {
  uint32_t c;
  asm("add.cc.u32 %0, %0, %5;\n\t"
      "addc.cc.u32 %1, %1, 0;\n\t"
      "addc.cc.u32 %2, %2, 0;\n\t"
      "addc.cc.u32 %3, %3, 0;\n\t"
      "addc.u32 %4, 0, 0;"
      : "+r"(s[0]), "+r"(s[1]), "+r"(s[2]), "+r"(s[3]), "=r"(c)
      : "r"(cin));
  return c;
}

template <int L>
BN_DEV void chunk_sum(const uint32_t (&x)[L], const uint32_t (&y)[L], uint32_t (&s)[L], uint32_t& g,
                      uint32_t& p, uint32_t cin = 0) {
  static_assert(L % 4 == 0, "L must be a multiple of 4");
  uint32_t c = cin, all = 0xFFFFFFFFu;
#pragma unroll
  for (int v = 0; v < L / 4; v++) {
    uint32_t t[4];
    c = add4_cc(t, x + 4 * v, y + 4 * v, c);
#pragma unroll
    for (int i = 0; i < 4; i++) {
      s[4 * v + i] = t[i];
      all &= t[i];
    }
  }
  g = c;
  p = all == 0xFFFFFFFFu;
}

// Step (3): r_i = p_i + carry_i — with s already the full
// chunk sum, the exclusive scan value at limb i is the chunk's carry-in
// rippled through s: one carry-chain increment (x is not needed).
template <int L>
BN_DEV void chunk_apply(const uint32_t (&x)[L], uint32_t (&s)[L], uint32_t cin) {
  (void)x;
#pragma unroll
  for (int v = 0; v < L / 4; v++) {
    uint32_t t[4] = {s[4 * v], s[4 * v + 1], s[4 * v + 2], s[4 * v + 3]};
    cin = inc4_cc(t, cin);
#pragma unroll
    for (int i = 0; i < 4; i++) s[4 * v + i] = t[i];
  }
}

// Exclusive carry scan across the TPI threads of each instance (steps (2)).
// Threads of one instance are consecutive (tid / TPI = instance slot).
// Every thread of the CTA must call this (it may contain __syncthreads when
// TPI > 32).  `agg` is shared scratch of >= blockDim.x / 32 words.
// Returns this thread's carry-in.
template <int TPI>
BN_DEV uint32_t carry_scan(uint32_t g, uint32_t p, uint32_t* agg) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t G = __ballot_sync(0xFFFFFFFFu, g);
  uint32_t P = __ballot_sync(0xFFFFFFFFu, p);
  if constexpr (TPI < 32) {
    constexpr uint32_t top = seg_top_mask<TPI>();
    G &= ~top;
    P &= ~top;
    uint32_t X = G | P;
    uint32_t cin = ((X + G) ^ X ^ G);
    return (cin >> lane) & 1u;
  } else {
    constexpr int WPI = TPI / 32;  // warps per instance
    uint32_t X = G | P;
    // warp aggregate: carry out of bit 31 with warp carry-in 0, and all-propagate
    uint64_t S = (uint64_t)X + G;
    const uint32_t warp = threadIdx.x >> 5;
    if constexpr (WPI > 1) {
      if (lane == 0) agg[warp] = (uint32_t)(S >> 32) | ((P == 0xFFFFFFFFu) << 1);
      __syncthreads();
      const uint32_t w0 = warp - (warp % WPI);  // first warp of my instance
      uint32_t a = lane < WPI ? agg[w0 + lane] : 0u;
      uint32_t G2 = __ballot_sync(0xFFFFFFFFu, a & 1u);
      uint32_t P2 = __ballot_sync(0xFFFFFFFFu, (a >> 1) & 1u);
      uint32_t X2 = G2 | P2;
      uint32_t c0 = (((X2 + G2) ^ X2 ^ G2) >> (warp % WPI)) & 1u;
      uint32_t cin = (X + G + c0) ^ X ^ G;
      return (cin >> lane) & 1u;
    } else {
      uint32_t cin = ((X + G) ^ X ^ G);
      return (cin >> lane) & 1u;
    }
  }
}

// ------------------------------------------------------- DSMEM primitives
// 32-bit shared::cluster addressing (half the registers of generic pointers):
// the address of `p` (this CTA's shared memory) in CTA `rank` of the cluster.
BN_DEV uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
BN_DEV uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
BN_DEV void st_cluster(uint32_t caddr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(caddr), "r"(v) : "memory");
}

// ------------------------------------------------------- cluster carry scan
// One instance spread over the CR CTAs of a thread-block cluster (sizes
// beyond one CTA): CTA rank r holds the r-th contiguous
// slice of the limbs, every CTA has the same number (<= 1024) of threads.  Three levels of the same
// carry operator (hierarchical as in PAPER.md:289-292):
// lanes (ballot-add), warps (ballot-add over the 32 warp aggregates), CTAs
// (each CTA's aggregate is written into every CTA's shared memory through
// DSMEM, then folded sequentially: CR <= 16).  The carry into the CTA enters
// the warp-level ballot-add as its initial carry.  cta_agg: CR words of
// shared memory per buffer, double-buffered by `parity` so consecutive
// instances need one cluster barrier each.  Every thread of every CTA of the
// cluster must call it, and the caller must have passed one cluster barrier
// since the kernel started before the first call (the remote stores below
// may only target CTAs that are already running).
template <int CR, class Cluster>
BN_DEV uint32_t cluster_carry_scan(uint32_t g, uint32_t p, uint32_t* agg, uint32_t* cta_agg, int parity,
                                   Cluster& cl) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t G = __ballot_sync(0xFFFFFFFFu, g);
  const uint32_t P = __ballot_sync(0xFFFFFFFFu, p);
  const uint32_t X = G | P;
  if (lane == 0) agg[warp] = (uint32_t)(((uint64_t)X + G) >> 32) | ((P == 0xFFFFFFFFu) << 1);
  __syncthreads();
  // warp aggregates; lanes past the CTA's warp count hold the operator's
  // identity (g = 0, p = 1), which leaves the CTA aggregate unchanged
  const uint32_t a = lane < (blockDim.x >> 5) ? agg[lane] : 2u;
  const uint32_t G2 = __ballot_sync(0xFFFFFFFFu, a & 1u);
  const uint32_t P2 = __ballot_sync(0xFFFFFFFFu, (a >> 1) & 1u);
  const uint32_t X2 = G2 | P2;
  const unsigned rank = cl.block_rank();
  uint32_t* buf = cta_agg + parity * CR;
  if (threadIdx.x < CR) {
    // this CTA's aggregate into slot `rank` of CTA threadIdx.x (DSMEM)
    const uint32_t v = (uint32_t)(((uint64_t)X2 + G2) >> 32) | ((P2 == 0xFFFFFFFFu) << 1);
    st_cluster(mapa_rank(smem_addr(buf + rank), threadIdx.x), v);
  }
  cl.sync();
  uint32_t c_cta = 0;
  for (unsigned r = 0; r < rank; r++) {
    const uint32_t v = buf[r];
    c_cta = (v & 1u) | ((v >> 1) & c_cta);
  }
  const uint32_t c0 = (((X2 + G2 + c_cta) ^ X2 ^ G2) >> warp) & 1u;
  return (((X + G + c0) ^ X ^ G) >> lane) & 1u;
}

// r = x + y over an instance whose L*TPI limbs are spread over TPI
// consecutive threads (thread k holds limbs [k*L, (k+1)*L)); valid == false
// threads contribute kill and their result is garbage (not stored).
template <int L, int TPI>
BN_DEV void add_regs(const uint32_t (&x)[L], const uint32_t (&y)[L], uint32_t (&r)[L], bool valid,
                     uint32_t* agg) {
  uint32_t g, p;
  chunk_sum<L>(x, y, r, g, p);
  if (!valid) g = p = 0;
  uint32_t cin = carry_scan<TPI>(g, p, agg);
  chunk_apply<L>(x, r, cin);
}

// Carry-save chaining of consecutive additions r_k = r_{k-1} + z_k (the
// fused 6-Add): addition k is left pending as (s, cin, p) — the chunk sum,
// the chunk's carry-in from its scan, the chunk's all-ones flag — and its
// final increment r_k = s + cin is folded into the NEXT addition's carry
// chain as that chain's carry-in, so every addition but the last costs one
// L-limb carry chain instead of two.  The fold counts a carry twice in one
// case only: s all ones and cin = 1 (r_k's chunk is 0, its carry already
// went to the chunk above through addition k's scan); then the next chain's
// carry-out is cleared.  Each addition is still a full §2 carry scan.
template <int L, int TPI>
BN_DEV void add_pending(uint32_t (&s)[L], const uint32_t (&z)[L], uint32_t& cin, uint32_t& p, bool valid,
                        uint32_t* agg) {
  const uint32_t ov = p & cin;
  uint32_t g;
  chunk_sum<L>(s, z, s, g, p, cin);
  g &= ~ov;
  if (!valid) g = p = 0;
  cin = carry_scan<TPI>(g, p, agg);
}

// r += y in place (the fused 6-Add accumulator: one limb set fewer live
// than add_regs).
template <int L, int TPI>
BN_DEV void add_regs_inplace(uint32_t (&r)[L], const uint32_t (&y)[L], bool valid, uint32_t* agg) {
  uint32_t g, p;
  chunk_sum<L>(r, y, r, g, p);
  if (!valid) g = p = 0;
  uint32_t cin = carry_scan<TPI>(g, p, agg);
  chunk_apply<L>(y, r, cin);
}

}  // namespace bn
