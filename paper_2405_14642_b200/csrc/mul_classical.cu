// mul_classical.cu — bn_mul_classical: quadratic multiplication, truncated.
//
// C_k = sum_{i+j=k, 0<=i,j,k<M} A_i B_j  (Eq. 1), with the
// paper's load-balanced result partitioning (Fig. 5): a
// thread owns the Q-column chunk starting at k1 = Q*g AND its mirror chunk
// starting at k1' = M - Q*(g+1), so every thread forms ~Q*(M+Q) partial
// products.  Per chunk (Fig. 7 `convolution`) the Q column
// sums are accumulated in registers as 96-bit (lo, hi, top) values; `combine`
// folds them into Q low words + high + carry; the results
// are published into shared arrays L and H (Fig. 6 step 3, PAPER.md:498-500;
// layout = DESIGN.md reading R8) and resolved by one scan-add R = L + H
// (reusing the §2 carry scan).
//
// B200 specifics:
//  * the column update is a u32 mad.lo.cc / madc.hi.cc / addc chain, which
//    ptxas lowers to one IMAD.WIDE.U32 (with carry-out predicate) plus half an
//    IADD3.X per 32x32 partial product — the kernel is bound by IMAD.WIDE
//    issue on the FMA pipe (32 lanes/clk/SM measured, profiles/r01_int_peak);
//  * the B operand is consumed through a sliding register window: one
//    128-bit shared load of B and one broadcast 128-bit load of A per Q x Q
//    block of partial products (the paper's loop at PAPER.md:583-588 with the
//    triangle of PAPER.md:589-592 absorbed by a zero chunk in front of B);
//  * the two partitions run as two calls of the same uniform loop, and for
//    small sizes I instances are interleaved across the lanes of a warp so
//    that lanes of a warp have (nearly) the same trip count: divergence
//    overhead (C-1)Q/(M+Q) with C = 32/I column groups per warp (<= 3%).
#include <cooperative_groups.h>

#include "bn_common.cuh"
#include "bn_kernels.h"

namespace cg = cooperative_groups;


namespace bn {

BN_DEV void mac3(uint32_t& lo, uint32_t& hi, uint32_t& top, uint32_t a, uint32_t b) {
  asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
      "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
      "addc.u32 %2, %2, 0;"
      : "+r"(lo), "+r"(hi), "+r"(top)
      : "r"(a), "r"(b));
}

// 1024-thread CTA targets (A/B against 512, ms per paper batch): 1-Mul 8K
// 2.605 -> 2.516, 16K 5.09 -> 4.98, 32K 9.30 -> 9.20, 64K 18.73 -> 17.97
// (128K: 37.5 -> 39.0, so it stops there); Poly 32K 31.3 -> 30.5, 64K 60.4 ->
// 58.2, 128K 122.2 -> 112.7; the wide kernel gains nothing (64K: +9.6%).
constexpr int mul1_tt(int logm) { return logm >= 8 && logm <= BN_CLASSICAL_1024_MAXLOG ? 1024 : 0; }
constexpr int polyc_tt(int logm) { return logm >= 8 && logm <= BN_POLYC_1024_MAXLOG ? 1024 : 0; }

template <int LOGM, int Q_, int TTX = 0>
struct MulCCfg {
  static constexpr int M = 1 << LOGM;
  static constexpr int Q = Q_;
  static constexpr int G = M / (2 * Q);  // column-group threads per instance
  // instances interleaved across warp lanes (keeps trip counts uniform)
  // target threads per CTA: 128 at 1K bits (A/B vs 256: 1-Mul -4%, wide
  // -8%, Poly -8%; 64 is 28% slower), 256 at 2K (more, smaller CTAs overlap
  // one group's barriers / epilogue with another's convolution: -4% vs 512;
  // 128 is 27% slower), 512 above (256 is 10% slower at 4K)
  static constexpr int TT = BN_CLASSICAL_TT > 0 ? BN_CLASSICAL_TT
                            : TTX > 0 ? TTX : (LOGM == 5 ? BN_CLASSICAL_1K_TT : LOGM == 6 ? 256 : 512);
  static constexpr int I = (TT / G) >= 32 ? 32 : ((TT / G) < 1 ? 1 : TT / G);
  static constexpr int SET_T = I * G;                         // threads per instance set
  static constexpr int SETS = SET_T >= TT ? 1 : TT / SET_T;   // sets per CTA
  static constexpr int T = SETS * SET_T;                       // threads per CTA
  static constexpr int IPB = SETS * I;                         // instances per CTA
  static constexpr int SA = M + 4;  // A stride: SA/4 odd -> broadcast A loads of <= 8 instances hit distinct banks
  // B stride: Q zero words + M, padded so that SB/4 == BS (mod 8), which makes the
  // 128-bit window loads of the 8 lanes (inst_lo, g) of a quarter-warp conflict-free
  static constexpr int BS = I >= 8 ? 1 : 8 / I;
  static constexpr int SB = M + Q + (((4 * BS - Q) % 32) + 32) % 32;
  static constexpr int STAGE_WORDS = IPB * (SA + SB);      // one group's A and B
  static constexpr int SMEM_WORDS = 2 * STAGE_WORDS + T / 32;  // double-buffered
  static constexpr int MINB = T >= 1024 ? 1 : 1024 / T;  // target residency: 64 registers
  // the 1-Mul kernel at 2K bits: 6 CTAs (40 registers, no spills) by A/B
  // 0.777 -> 0.748 ms; at 1K the same costs 4% and 5 CTAs (48 registers)
  // costs 4%; the fused / wide kernels spill and lose 2-10% at either
  static constexpr int MINB1 = LOGM == 6 ? BN_CLASSICAL_2K_MINB : MINB;
  static_assert(Q >= 2 && (Q % 4) == 0, "Q must be a multiple of 4 (>= 2 for the L/H layout)");
  static_assert(G >= 1, "size too small for Q");
};

// One Q x Q block of partial products: column q gets A[i] * B[j] for the Q
// consecutive i of `av` and the window B[k1 + q - i] held in cur / prev.
template <int Q>
BN_DEV void mac_block(uint32_t (&lo)[Q], uint32_t (&hi)[Q], uint32_t (&top)[Q], const uint32_t (&av)[Q],
                      const uint32_t (&cur)[Q], const uint32_t (&prev)[Q]) {
#pragma unroll
  for (int s = 0; s < Q; s++) {
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int d = q - s;
      mac3(lo[q], hi[q], top[q], av[s], d >= 0 ? cur[d] : prev[Q + d]);
    }
  }
}

// Q column sums starting at column Q*j0 (Fig. 7 convolution + combine).
// Ash: instance A (A[i] at Ash[i]); Bsh: instance B with B[x] at Bsh[x],
// B[-Q..-1] == 0.  Block c covers i in [Q c, Q c + Q) against B chunks
// j0 - c (cur) and j0 - c - 1 (prev); two blocks per trip so the window
// registers swap roles instead of being copied.
// REV: the staged operands are the reversed ones of the wide product's high
// half (mul_wide_classical_kernel), whose column Q j0 + q is the original
// column 2M - 1 - Q j0 - q: combine then runs over q descending so lhcs is
// in ascending original order.
// U4: 4 blocks per loop trip instead of 2 — ptxas then needs fewer
// register-shuffling IMAD.MOVs on the FMA-heavy pipe (A/B on B200: 3-4%
// faster for the 1-Mul kernel up to 8K bits, 3% slower at 32K).
template <int Q, bool REV = false, bool U4 = false>
BN_DEV void conv_chunk(const uint32_t* Ash, const uint32_t* Bsh, int j0, uint32_t (&lhcs)[Q + 2]) {
  uint32_t lo[Q], hi[Q], top[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) lo[q] = hi[q] = top[q] = 0;
  uint32_t b0[Q], b1[Q], av[Q];
  lds_limbs<Q>(b0, Bsh + Q * j0);
  const uint32_t* ap = Ash;
  const uint32_t* bp = Bsh + Q * (j0 - 1);
  int c = j0 + 1;  // blocks left
  if constexpr (U4) {
#pragma unroll 1
    for (; c >= 4; c -= 4) {
      lds_limbs<Q>(av, ap);
      lds_limbs<Q>(b1, bp);
      mac_block<Q>(lo, hi, top, av, b0, b1);
      lds_limbs<Q>(av, ap + Q);
      lds_limbs<Q>(b0, bp - Q);
      mac_block<Q>(lo, hi, top, av, b1, b0);
      lds_limbs<Q>(av, ap + 2 * Q);
      lds_limbs<Q>(b1, bp - 2 * Q);
      mac_block<Q>(lo, hi, top, av, b0, b1);
      lds_limbs<Q>(av, ap + 3 * Q);
      lds_limbs<Q>(b0, bp - 3 * Q);
      mac_block<Q>(lo, hi, top, av, b1, b0);
      ap += 4 * Q;
      bp -= 4 * Q;
    }
    if (c >= 2) {
      lds_limbs<Q>(av, ap);
      lds_limbs<Q>(b1, bp);
      mac_block<Q>(lo, hi, top, av, b0, b1);
      lds_limbs<Q>(av, ap + Q);
      lds_limbs<Q>(b0, bp - Q);
      mac_block<Q>(lo, hi, top, av, b1, b0);
      ap += 2 * Q;
      bp -= 2 * Q;
      c -= 2;
    }
  } else {
#pragma unroll 1
    for (; c >= 2; c -= 2) {
      lds_limbs<Q>(av, ap);
      lds_limbs<Q>(b1, bp);
      mac_block<Q>(lo, hi, top, av, b0, b1);
      lds_limbs<Q>(av, ap + Q);
      lds_limbs<Q>(b0, bp - Q);
      mac_block<Q>(lo, hi, top, av, b1, b0);
      ap += 2 * Q;
      bp -= 2 * Q;
    }
  }
  if (c) {
    lds_limbs<Q>(av, ap);
    lds_limbs<Q>(b1, bp);
    mac_block<Q>(lo, hi, top, av, b0, b1);
  }
  // combine: accum = (lo, hi), carry = top
  constexpr int F = REV ? Q - 1 : 0;
  lhcs[0] = lo[F];
  uint32_t h_res = hi[F], c_res = top[F];
#pragma unroll
  for (int q = 1; q < Q; q++) {
    const int x = REV ? Q - 1 - q : q;
    const uint32_t l = lo[x], h = hi[x];
    lhcs[q] = l + h_res;
    h_res = h + (c_res + (lhcs[q] < l));
    c_res = top[x] + (h_res < h);
  }
  lhcs[Q] = h_res;
  lhcs[Q + 1] = c_res;
}

// Squaring variant of conv_chunk (Poly's a*a and b*b): C_k = 2 sum_{i<j}
// a_i a_j + [k even] a_{k/2}^2, so only the blocks with i < j are formed —
// about half of them.  For column chunk j0 the full blocks c < j0/2 have
// i < j everywhere, blocks c > j0/2 only i > j (their transposes), and the
// single boundary block c = floor(j0/2) is masked per (row s, column q) at
// compile time by the parity of j0 (even: 2s < q doubled, 2s = q diagonal;
// odd: 2s - q < Q doubled, 2s - q = Q diagonal).  Off-diagonal sums are
// doubled once at the end; diagonal squares (one per even column) go to
// their own 64-bit accumulators.  Bsh is the same operand staged in the B
// layout (zero prefix).
template <int Q, int PAR>
BN_DEV void mac_block_sqr_edge(uint32_t (&lo)[Q], uint32_t (&hi)[Q], uint32_t (&top)[Q], uint32_t (&dlo)[Q],
                               uint32_t (&dhi)[Q], const uint32_t (&av)[Q], const uint32_t (&cur)[Q],
                               const uint32_t (&prev)[Q]) {
#pragma unroll
  for (int s = 0; s < Q; s++) {
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int d = q - s;
      const int key = 2 * s - q - (PAR ? Q : 0);  // < 0: doubled, == 0: diagonal
      if (key < 0) {
        mac3(lo[q], hi[q], top[q], av[s], d >= 0 ? cur[d] : prev[Q + d]);
      } else if (key == 0) {
        uint32_t t = 0;
        mac3(dlo[q], dhi[q], t, av[s], d >= 0 ? cur[d] : prev[Q + d]);
      }
    }
  }
}

template <int Q>
BN_DEV void conv_chunk_sqr(const uint32_t* Ash, const uint32_t* Bsh, int j0, uint32_t (&lhcs)[Q + 2]) {
  uint32_t lo[Q], hi[Q], top[Q], dlo[Q], dhi[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) lo[q] = hi[q] = top[q] = dlo[q] = dhi[q] = 0;
  uint32_t b0[Q], b1[Q], av[Q];
  lds_limbs<Q>(b0, Bsh + Q * j0);
  const uint32_t* ap = Ash;
  const uint32_t* bp = Bsh + Q * (j0 - 1);
  const int cm = j0 >> 1;  // boundary block
  int c = cm;              // full blocks before it
#pragma unroll 1
  for (; c >= 2; c -= 2) {
    lds_limbs<Q>(av, ap);
    lds_limbs<Q>(b1, bp);
    mac_block<Q>(lo, hi, top, av, b0, b1);
    lds_limbs<Q>(av, ap + Q);
    lds_limbs<Q>(b0, bp - Q);
    mac_block<Q>(lo, hi, top, av, b1, b0);
    ap += 2 * Q;
    bp -= 2 * Q;
  }
  if (c) {  // one more full block: the window roles swap for the edge
    lds_limbs<Q>(av, ap);
    lds_limbs<Q>(b1, bp);
    mac_block<Q>(lo, hi, top, av, b0, b1);
    lds_limbs<Q>(av, ap + Q);
    lds_limbs<Q>(b0, bp - Q);
    if (j0 & 1) mac_block_sqr_edge<Q, 1>(lo, hi, top, dlo, dhi, av, b1, b0);
    else mac_block_sqr_edge<Q, 0>(lo, hi, top, dlo, dhi, av, b1, b0);
  } else {
    lds_limbs<Q>(av, ap);
    lds_limbs<Q>(b1, bp);
    if (j0 & 1) mac_block_sqr_edge<Q, 1>(lo, hi, top, dlo, dhi, av, b0, b1);
    else mac_block_sqr_edge<Q, 0>(lo, hi, top, dlo, dhi, av, b0, b1);
  }
  // column sums: 2 * (lo, hi, top) + (dlo, dhi)
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const uint32_t t2 = (top[q] << 1) | (hi[q] >> 31);
    const uint32_t t1 = (hi[q] << 1) | (lo[q] >> 31);
    const uint32_t t0 = lo[q] << 1;
    asm("add.cc.u32 %0, %3, %4;\n\taddc.cc.u32 %1, %5, %6;\n\taddc.u32 %2, %7, 0;"
        : "=r"(lo[q]), "=r"(hi[q]), "=r"(top[q])
        : "r"(t0), "r"(dlo[q]), "r"(t1), "r"(dhi[q]), "r"(t2));
  }
  lhcs[0] = lo[0];
  uint32_t h_res = hi[0], c_res = top[0];
#pragma unroll
  for (int q = 1; q < Q; q++) {
    const uint32_t l = lo[q], h = hi[q];
    lhcs[q] = l + h_res;
    h_res = h + (c_res + (lhcs[q] < l));
    c_res = top[q] + (h_res < h);
  }
  lhcs[Q] = h_res;
  lhcs[Q + 1] = c_res;
}

// Thread roles inside a CTA (see MulCCfg): the convolution mapping
// interleaves instances across warp lanes; the resolve mapping is
// instance-major with G consecutive threads per instance.
template <class C>
struct MulCRoles {
  int t, conv_slot, g, add_slot, chunk;
  BN_DEV MulCRoles() {
    t = threadIdx.x;
    const int set = t / C::SET_T;
    const int r = t % C::SET_T;
    conv_slot = set * C::I + (r % C::I);
    g = r / C::I;
    add_slot = t / C::G;
    chunk = t % C::G;
  }
};

// B[-Q..-1] = 0 for every instance slot of `n_stages` stage buffers (never
// overwritten: loads and H start at B[0]).
template <class C>
BN_DEV void zero_b_prefix(uint32_t* sm, int n_stages) {
  for (int v = threadIdx.x; v < n_stages * C::IPB * C::Q; v += C::T) {
    const int st = v / (C::IPB * C::Q), k = (v / C::Q) % C::IPB;
    sm[st * C::STAGE_WORDS + C::IPB * C::SA + k * C::SB + (v % C::Q)] = 0u;
  }
}

// Stage x, y of one instance group with cp.async:
// coalesced 16-byte copies global -> shared; slots k >= n_valid are
// zero-filled.  x, y point at the group's first instance (stride M words).
template <class C>
BN_DEV void stage_xy(uint32_t* As, const uint32_t* x, const uint32_t* y, uint64_t n_valid) {
  constexpr int VPI = C::M / 4;  // uint4 per instance operand
  uint32_t* Bs = As + C::IPB * C::SA;
  for (int v = threadIdx.x; v < C::IPB * VPI; v += C::T) {
    const int k = v / VPI, w = (v % VPI) * 4;
    const bool ok = (uint64_t)k < n_valid;
    const uint64_t off = ok ? (uint64_t)k * C::M + w : 0;
    cp_async16(As + k * C::SA + w, x + off, ok);
    cp_async16(Bs + k * C::SB + C::Q + w, y + off, ok);
  }
}

// Convolution (Fig. 7) of the staged group and the L/H publish (reading R8),
// L over the A area, H over the B area.  Ends with a CTA barrier.
template <class C, bool SQ = false>
BN_DEV void conv_publish(uint32_t* As, const MulCRoles<C>& ro) {
  constexpr int M = C::M, Q = C::Q;
  uint32_t* Bs = As + C::IPB * C::SA;
  // ---- convolution: low chunk j0 = g and mirror chunk j0' = M/Q - 1 - g
  uint32_t lh0[Q + 2], lh1[Q + 2];
  {
    const uint32_t* Ai = As + ro.conv_slot * C::SA;
    const uint32_t* Bi = Bs + ro.conv_slot * C::SB + Q;
    if constexpr (SQ) {
      conv_chunk_sqr<Q>(Ai, Bi, ro.g, lh0);
      conv_chunk_sqr<Q>(Ai, Bi, M / Q - 1 - ro.g, lh1);
    } else {
      conv_chunk<Q>(Ai, Bi, ro.g, lh0);
      conv_chunk<Q>(Ai, Bi, M / Q - 1 - ro.g, lh1);
    }
  }
  __syncthreads();
  // ---- publish (reading R8): L[k1+q] = low_q; H[k1+Q] = high; H[k1+Q+1] = carry;
  // H[k1+Q+2 .. k1+2Q) = 0; the top chunk zeroes H[0..Q) instead.
  {
    uint32_t* L = As + ro.conv_slot * C::SA;
    uint32_t* H = Bs + ro.conv_slot * C::SB + Q;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t* lh = h == 0 ? lh0 : lh1;
      const int j0 = h == 0 ? ro.g : M / Q - 1 - ro.g;
      const int k1 = Q * j0;
      uint32_t lows[Q], hs[Q];
#pragma unroll
      for (int q = 0; q < Q; q++) {
        lows[q] = lh[q];
        hs[q] = q == 0 ? lh[Q] : (q == 1 ? lh[Q + 1] : 0u);
      }
      sts_limbs<Q>(L + k1, lows);
      if (k1 + Q < M) {
        sts_limbs<Q>(H + k1 + Q, hs);
      } else {
        uint32_t z[Q];
#pragma unroll
        for (int q = 0; q < Q; q++) z[q] = 0;
        sts_limbs<Q>(H, z);
      }
    }
  }
  __syncthreads();
}

// Resolve R = L + H into this thread's 2Q limbs
// (resolve mapping: limbs [2Q chunk, 2Q chunk + 2Q) of instance add_slot).
template <class C>
BN_DEV void resolve_lh(const uint32_t* As, const MulCRoles<C>& ro, bool valid, uint32_t* agg,
                       uint32_t (&res)[2 * C::Q]) {
  constexpr int L2 = 2 * C::Q;
  const uint32_t* Bs = As + C::IPB * C::SA;
  uint32_t x[L2], y[L2];
  lds_limbs<L2>(x, As + ro.add_slot * C::SA + L2 * ro.chunk);
  lds_limbs<L2>(y, Bs + ro.add_slot * C::SB + C::Q + L2 * ro.chunk);
  add_regs<L2, C::G>(x, y, res, valid, agg);
}

// The 1-Mul kernel keeps its convolution / publish / resolve inline rather
// than calling the phase helpers above: the same code routed through the
// helpers compiles (ptxas register assignment) to a mirror-chunk loop with
// five extra IMAD.MOVs on the saturated FMA-heavy pipe, 4-5% slower
// (A/B on one B200, scripts/ab.sh).
template <int LOGM, int Q>
__global__ void __launch_bounds__(MulCCfg<LOGM, Q, mul1_tt(LOGM)>::T, MulCCfg<LOGM, Q, mul1_tt(LOGM)>::MINB1)
    mul_classical_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst) {
  using C = MulCCfg<LOGM, Q, mul1_tt(LOGM)>;
  constexpr int M = C::M;
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* agg = sm + 2 * C::STAGE_WORDS;  // T/32

  const int t = threadIdx.x;
  // convolution mapping: lane = inst_lo + I * g_lo (instance-fastest)
  const int set = t / C::SET_T;
  const int r = t % C::SET_T;
  const int conv_slot = set * C::I + (r % C::I);
  const int g = r / C::I;
  // resolve/store mapping: instance-major, G consecutive threads per instance
  const int add_slot = t / C::G;
  const int chunk = t % C::G;

  // B[-Q..-1] = 0 in both stages (never overwritten: loads and H start at B[0])
  for (int v = t; v < 2 * C::IPB * Q; v += C::T) {
    const int st = v / (C::IPB * Q), k = (v / Q) % C::IPB;
    sm[st * C::STAGE_WORDS + C::IPB * C::SA + k * C::SB + (v % Q)] = 0u;
  }
  // stage A, B of a group with cp.async: coalesced 16-byte
  // copies global -> shared, zero-filled past the last instance
  constexpr int VPI = M / 4;  // uint4 per instance operand
  auto issue = [&](uint64_t grp, int st) {
    uint32_t* As = sm + st * C::STAGE_WORDS;
    uint32_t* Bs = As + C::IPB * C::SA;
    const uint64_t i0 = grp * C::IPB;
    for (int v = t; v < C::IPB * VPI; v += C::T) {
      const int k = v / VPI, w = (v % VPI) * 4;
      const bool ok = i0 + k < n_inst;
      const uint64_t off = ok ? (i0 + k) * M + w : 0;
      cp_async16(As + k * C::SA + w, a + off, ok);
      cp_async16(Bs + k * C::SB + Q + w, b + off, ok);
    }
  };

  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  uint64_t grp = blockIdx.x;
  if (grp < n_groups) issue(grp, 0);
  cp_async_commit();
  for (int st = 0; grp < n_groups; grp += gridDim.x, st ^= 1) {
    // prefetch the next group into the other stage while this one computes
    if (grp + gridDim.x < n_groups) issue(grp + gridDim.x, st ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    uint32_t* As = sm + st * C::STAGE_WORDS;
    uint32_t* Bs = As + C::IPB * C::SA;
    const uint64_t inst0 = grp * C::IPB;

    // ---- convolution: low chunk j0 = g and mirror chunk j0' = M/Q - 1 - g
    uint32_t lh0[Q + 2], lh1[Q + 2];
    {
      const uint32_t* Ai = As + conv_slot * C::SA;
      const uint32_t* Bi = Bs + conv_slot * C::SB + Q;
      conv_chunk<Q, false, (LOGM <= 8)>(Ai, Bi, g, lh0);
      conv_chunk<Q, false, (LOGM <= 8)>(Ai, Bi, M / Q - 1 - g, lh1);
    }
    __syncthreads();

    // ---- publish (reading R8): L[k1+q] = low_q; H[k1+Q] = high; H[k1+Q+1] = carry;
    // H[k1+Q+2 .. k1+2Q) = 0; the top chunk zeroes H[0..Q) instead.
    {
      uint32_t* L = As + conv_slot * C::SA;
      uint32_t* H = Bs + conv_slot * C::SB + Q;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const uint32_t* lh = h == 0 ? lh0 : lh1;
        const int j0 = h == 0 ? g : M / Q - 1 - g;
        const int k1 = Q * j0;
        uint32_t lows[Q], hs[Q];
#pragma unroll
        for (int q = 0; q < Q; q++) {
          lows[q] = lh[q];
          hs[q] = q == 0 ? lh[Q] : (q == 1 ? lh[Q + 1] : 0u);
        }
        sts_limbs<Q>(L + k1, lows);
        if (k1 + Q < M) {
          sts_limbs<Q>(H + k1 + Q, hs);
        } else {
          uint32_t z[Q];
#pragma unroll
          for (int q = 0; q < Q; q++) z[q] = 0;
          sts_limbs<Q>(H, z);
        }
      }
    }
    __syncthreads();

    // ---- resolve R = L + H and store
    {
      constexpr int L2 = 2 * Q;
      const uint64_t inst = inst0 + add_slot;
      const bool valid = inst < n_inst;
      uint32_t x[L2], y[L2], res[L2];
      lds_limbs<L2>(x, As + add_slot * C::SA + L2 * chunk);
      lds_limbs<L2>(y, Bs + add_slot * C::SB + Q + L2 * chunk);
      add_regs<L2, C::G>(x, y, res, valid, agg);
      if (valid) store_limbs<L2>(out + inst * M + L2 * chunk, res);
    }
    __syncthreads();  // this stage is refilled two groups from now
  }
  cp_async_wait<0>();
}

// Poly (Table 2 caption): (a*a + b) * (b*b + b) + a*b
// mod 2^bits — four classical multiplications and three additions in ONE
// kernel (block-level fusion).  Every phase is one multiplication of the
// kernel above with the addition fused into its epilogue (a second scan-add
// on the resolved product); the three intermediates t1 = a^2 + b,
// t2 = b^2 + b, t3 = a b go to this CTA's private slice of the caller's
// workspace (L2-resident: it is rewritten group after group by the same
// CTA) and come back as the operands of the last phase.
//   phase 1: t1 = a*a + b    phase 2: t2 = b*b + b
//   phase 3: t3 = a*b        phase 4: out = t1*t2 + t3
template <class C, bool AWS, bool OWS, bool SQ = false>
BN_DEV void classical_phase(uint32_t* As, uint32_t* agg, const MulCRoles<C>& ro, const uint32_t* x,
                            const uint32_t* y, const uint32_t* addend, uint32_t* dst, uint64_t n_valid) {
  constexpr int Q = C::Q, M = C::M;
  stage_xy<C>(As, x, y, n_valid);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  conv_publish<C, SQ>(As, ro);
  const bool valid = (uint64_t)ro.add_slot < n_valid;
  const uint64_t off = (uint64_t)ro.add_slot * M + 2 * Q * ro.chunk;
  uint32_t res[2 * Q];
  resolve_lh<C>(As, ro, valid, agg, res);
  if (addend) {
    uint32_t ad[2 * Q], r2[2 * Q];
    if (valid) load_any<AWS, 2 * Q>(ad, addend + off);
    else {
#pragma unroll
      for (int i = 0; i < 2 * Q; i++) ad[i] = 0;
    }
    if constexpr (C::G > 32) __syncthreads();  // agg reuse
    add_regs<2 * Q, C::G>(res, ad, r2, valid, agg);
    if (valid) store_any<OWS, 2 * Q>(dst + off, r2);
  } else {
    if (valid) store_any<OWS, 2 * Q>(dst + off, res);
  }
  __syncthreads();  // dst visible to the next phase; As / agg free
}

template <int LOGM, int Q>
__global__ void __launch_bounds__(MulCCfg<LOGM, Q, polyc_tt(LOGM)>::T, MulCCfg<LOGM, Q, polyc_tt(LOGM)>::MINB)
    poly_classical_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                          uint32_t* ws) {
  using C = MulCCfg<LOGM, Q, polyc_tt(LOGM)>;
  constexpr int M = C::M;
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* agg = sm + C::STAGE_WORDS;  // T/32
  const MulCRoles<C> ro;
  zero_b_prefix<C>(sm, 1);
  // this CTA's workspace slice: t1 | t2 | t3, each IPB * M words
  uint32_t* t1 = ws + (uint64_t)blockIdx.x * 3 * C::IPB * M;
  uint32_t* t2 = t1 + C::IPB * M;
  uint32_t* t3 = t2 + C::IPB * M;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  for (uint64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const uint64_t i0 = grp * C::IPB;
    const uint64_t nv = n_inst - i0 < (uint64_t)C::IPB ? n_inst - i0 : (uint64_t)C::IPB;
    const uint32_t* ag = a + i0 * M;
    const uint32_t* bg = b + i0 * M;
    classical_phase<C, false, true, true>(sm, agg, ro, ag, ag, bg, t1, nv);  // squares: half
    classical_phase<C, false, true, true>(sm, agg, ro, bg, bg, bg, t2, nv);  // the blocks
    classical_phase<C, false, true>(sm, agg, ro, ag, bg, nullptr, t3, nv);
    classical_phase<C, true, false>(sm, agg, ro, t1, t2, t3, out + i0 * M, nv);
  }
}

// ------------------------------------------------------------ full product
// Wide (untruncated) product: out[k] = a[k] * b[k] as 2M
// limbs, C_k = sum_{i+j=k} A_i B_j for 0 <= k < 2M (Eq. 1 without the
// k < M truncation).  The low half is exactly the truncated kernel's work.
// The high half uses the mirror identity: with A''_i = A_{M-i} (A''_0 = 0)
// and B'_j = B_{M-1-j}, column K < M of the truncated A'' B' equals the
// original column 2M-1-K, so the same conv_chunk (with a reversed combine)
// computes it; Fig. 5's load balance carries over, each thread owning the
// chunk pairs (g, M/Q-1-g) of both halves.  L / H span 2M words (reading R8
// with M -> 2M) and one scan-add resolves 2M limbs.
template <int LOGM, int Q_>
struct MulWCfg {
  using B = MulCCfg<LOGM, Q_>;
  static constexpr int M = B::M, Q = Q_, G = B::G, I = B::I, SET_T = B::SET_T, T = B::T, IPB = B::IPB;
  static constexpr int SA = 2 * M + 4;  // A | A''   (L afterwards)
  // B region: Q zeros | B | Q zeros | B' ; H = [Q, Q + 2M) afterwards
  static constexpr int SB = 2 * M + 2 * Q + (((4 * B::BS - 2 * Q) % 32) + 32) % 32;
  static constexpr int STAGE_WORDS = IPB * (SA + SB);
  static constexpr int SMEM_WORDS = STAGE_WORDS + T / 32;
  static constexpr int MINB = B::MINB;
};

template <int LOGM, int Q>
__global__ void __launch_bounds__(MulWCfg<LOGM, Q>::T, MulWCfg<LOGM, Q>::MINB)
    mul_wide_classical_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst) {
  using C = MulWCfg<LOGM, Q>;
  constexpr int M = C::M;
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* As = sm;
  uint32_t* Bs = sm + C::IPB * C::SA;
  uint32_t* agg = sm + C::STAGE_WORDS;
  const int t = threadIdx.x;
  const int set = t / C::SET_T;
  const int r = t % C::SET_T;
  const int conv_slot = set * C::I + (r % C::I);
  const int g = r / C::I;
  const int add_slot = t / C::G;
  const int chunk = t % C::G;
  constexpr int VPI = M / 4;

  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  for (uint64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const uint64_t i0 = grp * C::IPB;
    // stage A -> As[k][0, M), B -> Bs[k][Q, Q + M)
    for (int v = t; v < C::IPB * VPI; v += C::T) {
      const int k = v / VPI, w = (v % VPI) * 4;
      const bool ok = i0 + k < n_inst;
      const uint64_t off = ok ? (i0 + k) * M + w : 0;
      cp_async16(As + k * C::SA + w, a + off, ok);
      cp_async16(Bs + k * C::SB + Q + w, b + off, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // mirrored copies: A''_i = A_{M-i} (A''_0 = 0) at As[M + i]; B'_j =
    // B_{M-1-j} at Bs[2Q + M + j]; zero prefixes Bs[0, Q) and Bs[Q+M, 2Q+M)
    for (int v = t; v < C::IPB * M; v += C::T) {
      const int k = v / M, i = v % M;
      uint32_t* Ak = As + k * C::SA;
      uint32_t* Bk = Bs + k * C::SB;
      Ak[M + i] = i == 0 ? 0u : Ak[M - i];
      Bk[2 * Q + M + i] = Bk[Q + M - 1 - i];
      if (i < Q) {
        Bk[i] = 0u;
        Bk[Q + M + i] = 0u;
      }
    }
    __syncthreads();

    // ---- convolution: low pair (A, B) and high pair (A'', B')
    uint32_t lh[4][Q + 2];
    {
      const uint32_t* Ai = As + conv_slot * C::SA;
      const uint32_t* Bi = Bs + conv_slot * C::SB + Q;
      conv_chunk<Q>(Ai, Bi, g, lh[0]);
      conv_chunk<Q>(Ai, Bi, M / Q - 1 - g, lh[1]);
      conv_chunk<Q, true>(Ai + M, Bi + M + Q, g, lh[2]);
      conv_chunk<Q, true>(Ai + M, Bi + M + Q, M / Q - 1 - g, lh[3]);
    }
    __syncthreads();
    // ---- publish over 2M columns: L = As[k][0, 2M), H = Bs[k][Q, Q + 2M)
    {
      uint32_t* L = As + conv_slot * C::SA;
      uint32_t* H = Bs + conv_slot * C::SB + Q;
#pragma unroll
      for (int h = 0; h < 4; h++) {
        const int j0 = (h & 1) == 0 ? g : M / Q - 1 - g;
        // low chunks start at Q j0; high K-chunk j0 covers original columns
        // [2M - Q (j0 + 1), 2M - Q j0)
        const int k1 = h < 2 ? Q * j0 : 2 * M - Q * (j0 + 1);
        uint32_t lows[Q], hs[Q];
#pragma unroll
        for (int q = 0; q < Q; q++) {
          lows[q] = lh[h][q];
          hs[q] = q == 0 ? lh[h][Q] : (q == 1 ? lh[h][Q + 1] : 0u);
        }
        sts_limbs<Q>(L + k1, lows);
        if (k1 + Q < 2 * M) {
          sts_limbs<Q>(H + k1 + Q, hs);
        } else {
          uint32_t z[Q];
#pragma unroll
          for (int q = 0; q < Q; q++) z[q] = 0;
          sts_limbs<Q>(H, z);
        }
      }
    }
    __syncthreads();
    // ---- resolve R = L + H over 2M limbs (4Q per thread) and store
    {
      constexpr int L4 = 4 * Q;
      const uint64_t inst = i0 + add_slot;
      const bool valid = inst < n_inst;
      uint32_t x[L4], y[L4], res[L4];
      lds_limbs<L4>(x, As + add_slot * C::SA + L4 * chunk);
      lds_limbs<L4>(y, Bs + add_slot * C::SB + Q + L4 * chunk);
      add_regs<L4, C::G>(x, y, res, valid, agg);
      if (valid) store_limbs<L4>(out + inst * 2 * M + L4 * chunk, res);
    }
    __syncthreads();
  }
}

template <int LOGM>
static cudaError_t launch_mulw_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                 cudaStream_t st, int n_sm) {
  constexpr int Q = 4;
  using C = MulWCfg<LOGM, Q>;
  constexpr size_t smem = C::SMEM_WORDS * sizeof(uint32_t);
  static LaunchCache cache;
  int per_sm = 0;
  cudaError_t e = resident_ctas(cache, mul_wide_classical_kernel<LOGM, Q>, C::T, smem, &per_sm);
  if (e != cudaSuccess) return e;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t cap = (uint64_t)n_sm * per_sm * 4;
  const unsigned grid = cap_grid((unsigned)(n_groups < cap ? n_groups : cap));
  mul_wide_classical_kernel<LOGM, Q><<<grid, C::T, smem, st>>>(out, a, b, n_inst);
  return cudaGetLastError();
}

template <int LOGM>
static cudaError_t launch_mulc_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                 cudaStream_t st, int n_sm) {
  constexpr int Q = 4;
  using C = MulCCfg<LOGM, Q, mul1_tt(LOGM)>;
  constexpr size_t smem = C::SMEM_WORDS * sizeof(uint32_t);
  static LaunchCache cache;
  int per_sm = 0;
  cudaError_t e = resident_ctas(cache, mul_classical_kernel<LOGM, Q>, C::T, smem, &per_sm);
  if (e != cudaSuccess) return e;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t cap = (uint64_t)n_sm * per_sm;  // persistent: one wave of resident CTAs
  const unsigned grid = cap_grid((unsigned)(n_groups < cap ? n_groups : cap));
  mul_classical_kernel<LOGM, Q><<<grid, C::T, smem, st>>>(out, a, b, n_inst);
  return cudaGetLastError();
}

// Poly: one resident wave of persistent CTAs (each owns one workspace slice).
template <int LOGM>
static cudaError_t poly_geom_t(uint64_t n_inst, int n_sm, unsigned* grid, uint64_t* ws_words) {
  constexpr int Q = 4;
  using C = MulCCfg<LOGM, Q, polyc_tt(LOGM)>;
  constexpr size_t smem = (C::STAGE_WORDS + C::T / 32) * sizeof(uint32_t);
  static LaunchCache cache;
  int per_sm = 0;
  cudaError_t e = resident_ctas(cache, poly_classical_kernel<LOGM, Q>, C::T, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  const uint64_t cap = (uint64_t)n_sm * per_sm;
  *grid = cap_grid((unsigned)(n_groups < cap ? n_groups : cap));
  *ws_words = (uint64_t)*grid * 3 * C::IPB * C::M;
  return cudaSuccess;
}

template <int LOGM>
static cudaError_t launch_polyc_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                  uint32_t* ws, uint64_t ws_words, cudaStream_t st, int n_sm) {
  constexpr int Q = 4;
  using C = MulCCfg<LOGM, Q, polyc_tt(LOGM)>;
  unsigned grid = 0;
  uint64_t need = 0;
  cudaError_t e = poly_geom_t<LOGM>(n_inst, n_sm, &grid, &need);
  if (e != cudaSuccess) return e;
  if (ws_words < need) return cudaErrorInvalidValue;
  constexpr size_t smem = (C::STAGE_WORDS + C::T / 32) * sizeof(uint32_t);
  poly_classical_kernel<LOGM, Q><<<grid, C::T, smem, st>>>(out, a, b, n_inst, ws);
  return cudaGetLastError();
}

#define BN_LOGM_SWITCH(F, ...)                      \
  switch (logm) {                                   \
    case 5: return F<5>(__VA_ARGS__);               \
    case 6: return F<6>(__VA_ARGS__);               \
    case 7: return F<7>(__VA_ARGS__);               \
    case 8: return F<8>(__VA_ARGS__);               \
    case 9: return F<9>(__VA_ARGS__);               \
    case 10: return F<10>(__VA_ARGS__);             \
    case 11: return F<11>(__VA_ARGS__);             \
    case 12: return F<12>(__VA_ARGS__);             \
    case 13: return F<13>(__VA_ARGS__);             \
    default: return cudaErrorInvalidValue;          \
  }

template <int M, bool WIDE>
static cudaError_t launch_mulc_t1(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                  cudaStream_t st, int n_sm);

cudaError_t launch_mul_wide_classical(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b,
                                      uint64_t n_inst, cudaStream_t st, int n_sm) {
#if BN_CLASSICAL_T1
  if (logm == 5) return launch_mulc_t1<32, true>(out, a, b, n_inst, st, n_sm);
#endif
#if BN_CLASSICAL_T1_WIDE_2K
  if (logm == 6) return launch_mulc_t1<64, true>(out, a, b, n_inst, st, n_sm);
#endif

  BN_LOGM_SWITCH(launch_mulw_t, out, a, b, n_inst, st, n_sm)
}

cudaError_t poly_classical_geometry(int logm, uint64_t n_inst, int n_sm, uint64_t* ws_words) {
  unsigned grid = 0;
  BN_LOGM_SWITCH(poly_geom_t, n_inst, n_sm, &grid, ws_words)
}

template <int M>
static cudaError_t launch_polyc_t1(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                   cudaStream_t st, int n_sm);

cudaError_t launch_poly_classical(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b,
                                  uint64_t n_inst, uint32_t* ws, uint64_t ws_words, cudaStream_t st,
                                  int n_sm) {
#if BN_CLASSICAL_T1
  if (logm == 5 || (BN_POLY_T1_2K && logm == 6)) {
    // the one-thread kernel keeps its intermediates in shared memory; the
    // workspace contract (size check) is kept identical for every size
    unsigned grid = 0;
    uint64_t need = 0;
    cudaError_t e = logm == 5 ? poly_geom_t<5>(n_inst, n_sm, &grid, &need) : poly_geom_t<6>(n_inst, n_sm, &grid, &need);
    if (e != cudaSuccess) return e;
    if (ws_words < need) return cudaErrorInvalidValue;
    return logm == 5 ? launch_polyc_t1<32>(out, a, b, n_inst, st, n_sm) : launch_polyc_t1<64>(out, a, b, n_inst, st, n_sm);
  }
#endif
  BN_LOGM_SWITCH(launch_polyc_t, out, a, b, n_inst, ws, ws_words, st, n_sm)
}

// ------------------------------------------------------------ beyond one CTA
// 2^19 bits (m = 16384): one instance per cluster of 2 CTAs
// x 1024 threads.  Every CTA stages the whole of A and B (64 KiB each) —
// every chunk pair needs both operands in full — and global thread
// g = rank * 1024 + tid runs the Fig. 5 chunk pair (g, M/Q - 1 - g) exactly
// as the one-CTA kernel (Q = 4, G = 2048).  After a cluster barrier (no CTA
// may overwrite a peer's A/B while it convolves) the L/H publish goes to the
// CTA owning those limbs (CTA r owns [r M/2, (r+1) M/2); a chunk's Q-word runs
// never straddle owners) through DSMEM, and the resolve is the cluster carry
// scan.  2^20 bits would need 256 KiB of operands per CTA: not supported.
struct MulClCfg {
  static constexpr int LOGM = 14, M = 1 << LOGM, Q = 4, T = 1024, CR = 2;
  static constexpr int MS = M / CR;          // limbs owned (and resolved) per CTA
  static constexpr int SA = M + 4;           // A | L (owned half)
  static constexpr int SB = M + 2 * Q;       // Q zeros | B, H (owned half) at +Q
  static constexpr int SMEM_WORDS = SA + SB + 32 + 2 * CR;
  static_assert(MS == 8 * T && M / (2 * Q) == CR * T, "cluster classical layout");
};

BN_DEV void st_cluster_v4(uint32_t caddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(caddr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

__global__ void __launch_bounds__(1024, 1)
    mul_classical_cluster_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst) {
  using C = MulClCfg;
  constexpr int M = C::M, Q = C::Q, MS = C::MS;
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* As = sm;
  uint32_t* Bs = sm + C::SA;  // B[x] at Bs[Q + x]
  uint32_t* agg = Bs + C::SB;
  uint32_t* cta_agg = agg + 32;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const int g = rank * C::T + tid;
  if (tid < Q) Bs[tid] = 0u;  // B[-Q..-1] = 0, never overwritten
  const uint64_t n_cl = gridDim.x / C::CR;
  int parity = 0;
  for (uint64_t inst = blockIdx.x / C::CR; inst < n_inst; inst += n_cl, parity ^= 1) {
    // stage A and B (each CTA its own copy; the peer's copy hits L2)
    const uint32_t* ai = a + inst * M;
    const uint32_t* bi = b + inst * M;
    for (int v = tid; v < M / 4; v += C::T) {
      cp_async16(As + 4 * v, ai + 4 * v, true);
      cp_async16(Bs + Q + 4 * v, bi + 4 * v, true);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // convolution: chunk pair (g, M/Q - 1 - g)
    uint32_t lh0[Q + 2], lh1[Q + 2];
    conv_chunk<Q>(As, Bs + Q, g, lh0);
    conv_chunk<Q>(As, Bs + Q, M / Q - 1 - g, lh1);
    cl.sync();  // every CTA is done reading its A / B: L / H may overwrite them
    // publish into the owner's L (A area) / H (B area + Q), local index
    const uint32_t la = smem_addr(As), ha = smem_addr(Bs + Q);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t* lh = h == 0 ? lh0 : lh1;
      const int k1 = Q * (h == 0 ? g : M / Q - 1 - g);
      st_cluster_v4(mapa_rank(la + 4 * (k1 % MS), k1 / MS), lh[0], lh[1], lh[2], lh[3]);
      const int kh = k1 + Q < M ? k1 + Q : 0;  // top chunk: zeroes H[0, Q)
      const uint32_t h0 = k1 + Q < M ? lh[Q] : 0u, h1 = k1 + Q < M ? lh[Q + 1] : 0u;
      st_cluster_v4(mapa_rank(ha + 4 * (kh % MS), kh / MS), h0, h1, 0u, 0u);
    }
    cl.sync();
    // resolve this CTA's limbs [rank MS + 8 tid, +8)
    uint32_t x[8], y[8], r[8], gg, pp;
    lds_limbs<8>(x, As + 8 * tid);
    lds_limbs<8>(y, Bs + Q + 8 * tid);
    chunk_sum<8>(x, y, r, gg, pp);
    const uint32_t cin = cluster_carry_scan<C::CR>(gg, pp, agg, cta_agg, parity, cl);
    chunk_apply<8>(x, r, cin);
    store_limbs<8>(out + inst * M + (uint64_t)rank * MS + 8 * tid, r);
    __syncthreads();  // L / H reads done before the next instance's staging
  }
}

static cudaError_t launch_mulc_cluster(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                       cudaStream_t st, int n_sm) {
  using C = MulClCfg;
  constexpr size_t smem = C::SMEM_WORDS * sizeof(uint32_t);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(C::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.gridDim = dim3(C::CR);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::CR;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static LaunchCache cache;
  int max_cl = 0;
  cudaError_t e = cached_query(cache, [&](int* o) {
    cudaError_t e1 = cudaFuncSetAttribute(mul_classical_cluster_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e1 != cudaSuccess) return e1;
    return cudaOccupancyMaxActiveClusters(o, mul_classical_cluster_kernel, &cfg);
  }, &max_cl);
  if (e != cudaSuccess) return e;
  if (max_cl < 1) return cudaErrorInvalidConfiguration;
  uint64_t n_cl = n_inst < (uint64_t)max_cl ? n_inst : (uint64_t)max_cl;
  n_cl = cap_grid((unsigned)n_cl);
  cfg.gridDim = dim3((unsigned)(n_cl * C::CR));
  e = cudaLaunchKernelEx(&cfg, mul_classical_cluster_kernel, out, a, b, n_inst);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ------------------------------------------------------------ one thread per instance
// 1K and 2K bits (M = 32, 64): the Fig. 5 partitioning at its limit
// Q = M / 2, where one thread owns all M columns, so there is nothing to
// publish or resolve: the
// thread keeps A and B in registers and walks the columns in order (product
// scanning), carrying the 96-bit accumulator (lo, hi, top) from column k into
// column k + 1 — the column sums of Eq. 1 with the carry
// resolved sequentially (the ripple of PAPER.md:125-134).  M (M + 1) / 2
// partial products per thread, no CTA barriers.  A warp's tile is read in
// full before its product is stored, and the next tile staged meanwhile
// holds other instances, so in-place calls (out == a or b) are safe.
// threads per CTA: 4 warps for the 1K 1-Mul (one 8 KiB stage each), else 2
// (the 1K full product with two stages, 2K with one 16 KiB stage per warp)
constexpr int kT1Threads = 128;

// Operands reach the registers through a per-warp shared-memory tile of 32
// instances (A | B, 8 KiB): cp.async copies tile i + 1 (coalesced 512-byte
// runs) while the warp multiplies tile i, so the warps of an SM do not all
// wait on HBM at once (loading straight into registers left the FMA pipe
// 55% busy, long-scoreboard stalls 17 per issue: ncu).  16-byte chunk c of
// row r sits at r * 8 + (c ^ (r & 7)): a quarter-warp reading chunk k of its
// 8 rows touches 8 distinct bank quads.
// tiles in flight per warp (cp.async stages of A | B); A/B at 1K (ms):
// 1-Mul 1 stage 0.348 / 2 stages 0.368, full product 0.697 / 0.635
constexpr int t1_stages(int m, bool wide) { return m == 32 && wide ? 2 : 1; }
constexpr int t1_threads(int m, bool wide) { return m == 32 && t1_stages(m, wide) == 1 ? kT1Threads : 64; }
constexpr int t1_minb(int m, bool wide) {
  return m == 32 && !wide ? BN_CLASSICAL_T1_MINB : (wide && m == 64 ? BN_CLASSICAL_T1_MINB_WIDE_2K : BN_CLASSICAL_T1_MINB_2K);
}
// WIDE: all 2M columns (the full product, bn_mul_wide_classical).
template <int M, bool WIDE>
__global__ void __launch_bounds__(t1_threads(M, WIDE), t1_minb(M, WIDE))
    mul_classical_t1_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst) {
  static_assert(M % 32 == 0, "row swizzle assumes a multiple of 8 chunks per row");
  constexpr int W = t1_threads(M, WIDE) / 32, CH = M / 4, NS = t1_stages(M, WIDE);
  __shared__ uint4 buf[W][NS][2][32 * CH];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t n_tiles = (n_inst + 31) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * W;
  // stage st holds tile number it (0, 1, ...) of this warp with it % NS == st;
  // one commit group per tile (empty past the end) keeps the wait counts uniform
  auto stage = [&](uint64_t tile, int st) {
    if (tile < n_tiles) {
      uint4* As = buf[wid][st][0];
      uint4* Bs = buf[wid][st][1];
      const uint4* ga = reinterpret_cast<const uint4*>(a) + tile * 32 * CH;
      const uint4* gb = reinterpret_cast<const uint4*>(b) + tile * 32 * CH;
#pragma unroll
      for (int j = 0; j < CH; j++) {
        const int idx = lane + 32 * j, r = idx / CH, c = idx % CH;
        const bool valid = tile * 32 + r < n_inst;
        cp_async16(As + r * CH + (c ^ (r & 7)), ga + idx, valid);
        cp_async16(Bs + r * CH + (c ^ (r & 7)), gb + idx, valid);
      }
    }
    cp_async_commit();
  };
  uint64_t tile = (uint64_t)blockIdx.x * W + wid;
#pragma unroll
  for (int k = 0; k < NS; k++) stage(tile + k * nw, k);
  for (int st = 0; tile < n_tiles; tile += nw, st = st + 1 == NS ? 0 : st + 1) {
    uint32_t x[M], y[M];
    cp_async_wait<NS - 1>();
    __syncwarp();
    const uint4* As = buf[wid][st][0];
    const uint4* Bs = buf[wid][st][1];
#pragma unroll
    for (int v = 0; v < CH; v++) {
      const uint4 u = As[lane * CH + (v ^ (lane & 7))], w = Bs[lane * CH + (v ^ (lane & 7))];
      x[4 * v] = u.x; x[4 * v + 1] = u.y; x[4 * v + 2] = u.z; x[4 * v + 3] = u.w;
      y[4 * v] = w.x; y[4 * v + 1] = w.y; y[4 * v + 2] = w.z; y[4 * v + 3] = w.w;
    }
    __syncwarp();  // every lane has its row before the stage is refilled
    stage(tile + NS * nw, st);
    constexpr int MO = WIDE ? 2 * M : M;  // output limbs
    const uint64_t inst = tile * 32 + lane;
    uint4* o4 = reinterpret_cast<uint4*>(out + inst * MO);
    const bool valid = inst < n_inst;
    uint32_t lo = 0, hi = 0, top = 0, r[4];
#pragma unroll
    for (int k = 0; k < M; k++) {
#pragma unroll
      for (int i = 0; i <= k; i++) mac3(lo, hi, top, x[i], y[k - i]);
      r[k & 3] = lo;
      lo = hi;
      hi = top;
      top = 0;
      if ((k & 3) == 3 && valid) o4[k / 4] = make_uint4(r[0], r[1], r[2], r[3]);
    }
    if constexpr (WIDE) {
      // upper columns in two loop nests (one nest of M columns does not
      // unroll at M = 64, and the operand arrays would go to the stack)
#pragma unroll
      for (int k = M; k < 3 * M / 2; k++) {
#pragma unroll
        for (int i = k - M + 1; i < M; i++) mac3(lo, hi, top, x[i], y[k - i]);
        r[k & 3] = lo;
        lo = hi;
        hi = top;
        top = 0;
        if ((k & 3) == 3 && valid) o4[k / 4] = make_uint4(r[0], r[1], r[2], r[3]);
      }
#pragma unroll
      for (int k = 3 * M / 2; k < 2 * M; k++) {
#pragma unroll
        for (int i = k - M + 1; i < M; i++) mac3(lo, hi, top, x[i], y[k - i]);
        r[k & 3] = lo;
        lo = hi;
        hi = top;
        top = 0;
        if ((k & 3) == 3 && valid) o4[k / 4] = make_uint4(r[0], r[1], r[2], r[3]);
      }
    }
  }
}

template <int M, bool WIDE>
static cudaError_t launch_mulc_t1(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                  cudaStream_t st, int n_sm) {
  static LaunchCache cache;
  int per_sm = 0;
  cudaError_t e = resident_ctas(cache, mul_classical_t1_kernel<M, WIDE>, t1_threads(M, WIDE), 0, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  // persistent: one wave of CTAs, each warp walks its tiles
  const uint64_t need = (n_inst + t1_threads(M, WIDE) - 1) / t1_threads(M, WIDE);
  const uint64_t cap = (uint64_t)n_sm * per_sm;
  const unsigned grid = cap_grid((unsigned)(need < cap ? need : cap));
  mul_classical_t1_kernel<M, WIDE><<<grid, t1_threads(M, WIDE), 0, st>>>(out, a, b, n_inst);
  return cudaGetLastError();
}

// ------------------------------------------------------------ Poly, one thread per instance
// (a a + b)(b b + b) + a b mod 2^(32 M) on the 1K / 2K-bit
// one-thread-per-instance layout: four product scans, each addition folded
// into the column accumulator of the product that precedes it (column k of
// a a + b adds b_k before its low word is taken — the block-level fusion of
// P:988-991 at register level).  a a and b b are squaring scans: the
// off-diagonal column sum is formed once and doubled (272 instead of 528
// partial products).  a b and a a + b go to this warp's shared rows, b b + b
// stays in registers, then (a a + b)(b b + b) + a b streams to HBM.
constexpr int kPolyT1Threads = 64;  // 2 warps x 16 KiB of shared rows per CTA

BN_DEV void acc_add3(uint32_t& lo, uint32_t& hi, uint32_t& top, uint32_t c0, uint32_t c1, uint32_t c2) {
  asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
      : "+r"(lo), "+r"(hi), "+r"(top)
      : "r"(c0), "r"(c1), "r"(c2));
}

// Column k of x * y (SQ: x * x, y ignored) into the running accumulator.
template <int M, bool SQ>
BN_DEV void t1_column(const uint32_t (&x)[M], const uint32_t (&y)[M], int k, uint32_t& lo, uint32_t& hi,
                      uint32_t& top) {
  if constexpr (!SQ) {
#pragma unroll
    for (int i = 0; i <= k; i++) mac3(lo, hi, top, x[i], y[k - i]);
  } else {
    uint32_t s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
    for (int i = 0; 2 * i < k; i++) mac3(s0, s1, s2, x[i], x[k - i]);
    s2 = __funnelshift_l(s1, s2, 1);
    s1 = __funnelshift_l(s0, s1, 1);
    s0 <<= 1;
    if (k % 2 == 0) mac3(s0, s1, s2, x[k / 2], x[k / 2]);
    acc_add3(lo, hi, top, s0, s1, s2);
  }
}

// row helpers: 16-byte chunk c of row r at r * CH + (c ^ (r & 7))
template <int CH>
BN_DEV void row_store4(uint4* rows, int r, int c, const uint32_t (&v)[4]) {
  rows[r * CH + (c ^ (r & 7))] = make_uint4(v[0], v[1], v[2], v[3]);
}

// Columns [K0, K1) of x * y (SQ: x * x): add(k, lo, hi, top) folds an addend
// into column k, sink(k, lo) takes its low word.
template <int M, bool SQ, int K0, int K1, class Add, class Sink>
BN_DEV void t1_cols(const uint32_t (&x)[M], const uint32_t (&y)[M], uint32_t& lo, uint32_t& hi, uint32_t& top,
                    Add add, Sink sink) {
#pragma unroll
  for (int k = K0; k < K1; k++) {
    t1_column<M, SQ>(x, y, k, lo, hi, top);
    add(k, lo, hi, top);
    sink(k, lo);
    lo = hi;
    hi = top;
    top = 0;
  }
}
// the M columns of one truncated product; at M = 64 as two loop nests (one
// nest does not unroll and the operand arrays would go to the stack)
template <int M, bool SQ, class Add, class Sink>
BN_DEV void t1_prod(const uint32_t (&x)[M], const uint32_t (&y)[M], Add add, Sink sink) {
  uint32_t lo = 0, hi = 0, top = 0;
  if constexpr (M <= 32) {
    t1_cols<M, SQ, 0, M>(x, y, lo, hi, top, add, sink);
  } else {
    t1_cols<M, SQ, 0, M / 2>(x, y, lo, hi, top, add, sink);
    t1_cols<M, SQ, M / 2, M>(x, y, lo, hi, top, add, sink);
  }
}

// 2K (M = 64): the operand tile alone is 16 KiB per warp, so a b and a a + b
// overwrite it (each lane its own rows) and the next tile is loaded after
// the product instead of during it (PF = false).
template <int M>
__global__ void __launch_bounds__(kPolyT1Threads, M == 32 ? BN_POLY_T1_MINB : BN_POLY_T1_MINB_2K)
    poly_classical_t1_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst) {
  static_assert(M % 32 == 0, "row swizzle assumes a multiple of 8 chunks per row");
  constexpr bool PF = M == 32;
  constexpr int W = kPolyT1Threads / 32, CH = M / 4, NB = PF ? 4 : 2;
  __shared__ uint4 buf[W][NB][32 * CH];  // A tile | B tile [| a b | a a + b]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint4* As = buf[wid][0];
  uint4* Bs = buf[wid][1];
  uint4* T3 = buf[wid][PF ? 2 : 0];
  uint4* T1 = buf[wid][PF ? 3 : 1];
  const uint64_t n_tiles = (n_inst + 31) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * W;
  auto stage = [&](uint64_t tile) {
    const uint4* ga = reinterpret_cast<const uint4*>(a) + tile * 32 * CH;
    const uint4* gb = reinterpret_cast<const uint4*>(b) + tile * 32 * CH;
#pragma unroll
    for (int j = 0; j < CH; j++) {
      const int idx = lane + 32 * j, r = idx / CH, c = idx % CH;
      const bool valid = tile * 32 + r < n_inst;
      cp_async16(As + r * CH + (c ^ (r & 7)), ga + idx, valid);
      cp_async16(Bs + r * CH + (c ^ (r & 7)), gb + idx, valid);
    }
    cp_async_commit();
  };
  auto load_row = [&](const uint4* rows, uint32_t(&v)[M]) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      const uint4 u = rows[lane * CH + (c ^ (lane & 7))];
      v[4 * c] = u.x; v[4 * c + 1] = u.y; v[4 * c + 2] = u.z; v[4 * c + 3] = u.w;
    }
  };
  uint64_t tile = (uint64_t)blockIdx.x * W + wid;
  if (PF && tile < n_tiles) stage(tile);
  for (; tile < n_tiles; tile += nw) {
    uint32_t x[M], y[M];
    if constexpr (!PF) {
      __syncwarp();  // every lane is done with its rows of the previous tile
      stage(tile);
    }
    cp_async_wait<0>();
    __syncwarp();
    load_row(As, x);
    load_row(Bs, y);
    __syncwarp();
    if (PF && tile + nw < n_tiles) stage(tile + nw);
    const uint64_t inst = tile * 32 + lane;
    const bool valid = inst < n_inst;
    uint32_t r[4];
    auto none = [](int, uint32_t&, uint32_t&, uint32_t&) {};
    auto plus_b = [&](int k, uint32_t& lo, uint32_t& hi, uint32_t& top) { acc_add3(lo, hi, top, y[k], 0u, 0u); };
    // t3 = a b -> T3
    t1_prod<M, false>(x, y, none, [&](int k, uint32_t lo) {
      r[k & 3] = lo;
      if ((k & 3) == 3) row_store4<CH>(T3, lane, k / 4, r);
    });
    // t1 = a a + b -> T1
    t1_prod<M, true>(x, x, plus_b, [&](int k, uint32_t lo) {
      r[k & 3] = lo;
      if ((k & 3) == 3) row_store4<CH>(T1, lane, k / 4, r);
    });
    // t2 = b b + b -> registers (x is free: it takes t2)
    t1_prod<M, true>(y, y, plus_b, [&](int k, uint32_t lo) { x[k] = lo; });
    // out = t1 t2 + t3 (own rows only: no barrier needed)
    load_row(T1, y);
    uint4* o4 = reinterpret_cast<uint4*>(out + inst * M);
    t1_prod<M, false>(y, x, [&](int k, uint32_t& lo, uint32_t& hi, uint32_t& top) {
      if ((k & 3) == 0) {
        const uint4 u = T3[lane * CH + ((k / 4) ^ (lane & 7))];
        r[0] = u.x; r[1] = u.y; r[2] = u.z; r[3] = u.w;
      }
      acc_add3(lo, hi, top, r[k & 3], 0u, 0u);
    }, [&](int k, uint32_t lo) {
      r[k & 3] = lo;
      if ((k & 3) == 3 && valid) o4[k / 4] = make_uint4(r[0], r[1], r[2], r[3]);
    });
  }
}

template <int M>
static cudaError_t launch_polyc_t1(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                   cudaStream_t st, int n_sm) {
  static LaunchCache cache;
  int per_sm = 0;
  cudaError_t e = resident_ctas(cache, poly_classical_t1_kernel<M>, kPolyT1Threads, 0, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t need = (n_inst + kPolyT1Threads - 1) / kPolyT1Threads;
  const uint64_t cap = (uint64_t)n_sm * per_sm;
  const unsigned grid = cap_grid((unsigned)(need < cap ? need : cap));
  poly_classical_t1_kernel<M><<<grid, kPolyT1Threads, 0, st>>>(out, a, b, n_inst);
  return cudaGetLastError();
}

cudaError_t launch_mul_classical(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b,
                                 uint64_t n_inst, cudaStream_t st, int n_sm) {
  switch (logm) {
#if BN_CLASSICAL_T1
    case 5: return launch_mulc_t1<32, false>(out, a, b, n_inst, st, n_sm);
#else
    case 5: return launch_mulc_t<5>(out, a, b, n_inst, st, n_sm);
#endif
#if BN_CLASSICAL_T1_2K
    case 6: return launch_mulc_t1<64, false>(out, a, b, n_inst, st, n_sm);
#else
    case 6: return launch_mulc_t<6>(out, a, b, n_inst, st, n_sm);
#endif
    case 7: return launch_mulc_t<7>(out, a, b, n_inst, st, n_sm);
    case 8: return launch_mulc_t<8>(out, a, b, n_inst, st, n_sm);
    case 9: return launch_mulc_t<9>(out, a, b, n_inst, st, n_sm);
    case 10: return launch_mulc_t<10>(out, a, b, n_inst, st, n_sm);
    case 11: return launch_mulc_t<11>(out, a, b, n_inst, st, n_sm);
    case 12: return launch_mulc_t<12>(out, a, b, n_inst, st, n_sm);
    case 13: return launch_mulc_t<13>(out, a, b, n_inst, st, n_sm);
    case 14: return launch_mulc_cluster(out, a, b, n_inst, st, n_sm);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bn
