// mul_ntt.cu — bn_mul_ntt: exact FFT multiplication over word-size primes.
//
// The paper's §4: transform A and B over a prime field
// Z_p with p = k 2^n + 1, multiply pointwise, transform
// back, then resolve the carries by a scan-add (bmulFFT, Fig. 9,
// PAPER.md:767-788, splitFftReg/publish PAPER.md:816-821).  The printed
// digit scheme is inexact (readings R10/R11), so this kernel uses
// the exact variant: the u32 limbs ARE the digits, both operands are
// zero-padded to N = 2m points, and three primes p0 < p1 < p2 < 2^30 with
// Garner CRT recover every coefficient c_k <= m (2^32-1)^2 < 2^77 < p0 p1 p2.
//
// One instance per TPI = N/16 threads (IPB instances per CTA); each thread
// holds R = 16 elements in registers and performs 4 radix-2 stages per
// register pass; passes exchange through a shared buffer X with an XOR
// swizzle that makes every pass's access pattern bank-conflict free.
//   forward  : DIF (Gentleman–Sande), natural in -> bit-reversed out,
//              Harvey-lazy values in [0, 2p), Shoup twiddle products;
//   pointwise: Montgomery product (R = 2^32), values stay in [0, 2p);
//   inverse  : DIT (Cooley–Tukey) with omega^-1, bit-reversed in -> natural
//              out, values in [0, 4p); 1/N and R are folded into the CRT
//              constants (PAPER.md:764's "scale by invM" moved into Garner).
// Because the DIF output order is exactly the DIT input order, no bit
// reversal is ever performed, and the last forward pass / pointwise product
// / first inverse pass happen in registers without a shared-memory trip.
// Per thread, then, 8 consecutive coefficients are CRT'd and aggregated into
// 8 low words + 2 overflow words (< 2^46), published into L/H exactly like
// the classical kernel (reading R8) and resolved by the §2 scan-add.
#include <cooperative_groups.h>

#include "bn_common.cuh"
#include "bn_kernels.h"

namespace cg = cooperative_groups;

// Kernel geometry (CTA sizes, residency targets, which layout runs at which
// size) is one table with its A/B evidence: bn_config.h.
// CTA target of the 16-element Poly kernel
constexpr int kPolyNttTT = BN_POLY_NTT_TT;
// Timing-only experiment (never in a shipped build): BN_DBG_TWCONST replaces
// every twiddle load by a value derived from the pointer (no memory access),
// to measure what the table loads cost.  Results are WRONG with it.
#ifdef BN_DBG_TWCONST
#define BN_DBG_TW(ptr) make_uint2((uint32_t)(uintptr_t)(ptr) & 0x3FFFFFFu, 0x5u)
#else
#define BN_DBG_TW(ptr) __ldg(ptr)
#endif


namespace bn {

__constant__ PrimeConst c_pc[kNumPrimes];
__constant__ CrtConst c_crt[kMaxLogN + 1];

cudaError_t upload_prime_consts(const PrimeConst (&pc)[kNumPrimes], const CrtConst (&crt)[kMaxLogN + 1]) {
  cudaError_t e = cudaMemcpyToSymbol(c_pc, pc, sizeof(pc));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_crt, crt, sizeof(crt));
}

// ------------------------------------------------------------ field arithmetic
// Shoup: w < p, wsh = floor(w 2^32 / p); any x < 2^32 -> x w mod p in [0, 2p).
BN_DEV uint32_t shoup(uint32_t x, uint32_t w, uint32_t wsh, uint32_t p) {
  const uint32_t q = __umulhi(x, wsh);
  return x * w - q * p;
}
// x < 2m -> x mod m (one VIADDMNMX: min(x, x - m) as unsigned)
BN_DEV uint32_t red2(uint32_t x, uint32_t m) { return min(x, x - m); }
// Montgomery: a, b < 2p, p < 2^30 -> a b 2^-32 mod p in [0, 2p)
BN_DEV uint32_t mont(uint32_t a, uint32_t b, uint32_t p, uint32_t pinv) {
  const uint64_t t = (uint64_t)a * b;
  const uint32_t m = (uint32_t)t * pinv;
  const uint64_t u = t + (uint64_t)m * p;
  return (uint32_t)(u >> 32);
}
// DIF butterfly, inputs [0, 2p) -> outputs [0, 2p)
BN_DEV void gs_bfly(uint32_t& x, uint32_t& y, uint2 w, uint32_t p, uint32_t p2) {
  const uint32_t s = x + y;
  const uint32_t d = x - y + p2;
  x = red2(s, p2);
  y = shoup(d, w.x, w.y, p);
}
// DIT butterfly, inputs [0, 4p) -> outputs [0, 4p)
BN_DEV void ct_bfly(uint32_t& x, uint32_t& y, uint2 w, uint32_t p, uint32_t p2) {
  const uint32_t u = red2(x, p2);
  const uint32_t v = shoup(y, w.x, w.y, p);
  x = u + v;
  y = u - v + p2;
}

// ------------------------------------------------------------ layout
template <int LOGN, int TTA = BN_NTT_TT>
struct NttCfg {
  static constexpr int N = 1 << LOGN;
  static constexpr int M = N / 2;
  static constexpr int R = 16;
  static constexpr int TPI = N / R;
  static constexpr int NP = (LOGN + 3) / 4;  // register passes
  static constexpr int TT = LOGN <= BN_NTT_TT_MAXLOG ? TTA : 256;  // target threads per CTA
  static constexpr int IPB = TPI >= TT ? 1 : TT / TPI;
  static constexpr int T = IPB * TPI;
  // exchange area (padded by 1/16 for LOGN <= 8, see xbase), raw residues, agg
  static constexpr int XW = LOGN <= 8 ? IPB * N + (IPB * N >> 4) : IPB * N;
  // two exchange planes (A and B are transformed together), raw residues, agg
  static constexpr int SMEM_WORDS = 2 * XW + IPB * (3 * M + (TPI < 32 ? 16 : 0)) + T / 32;
  // residency (threads per SM) for 2^9 .. 2^12 points (bn_config.h): 768 at
  // 2^12, BN_NTT_MID9_THREADS at 2^9, 512 between
  static constexpr int MT = LOGN >= BN_NTT_MID768_MINLOG ? 768 : (LOGN == 9 ? BN_NTT_MID9_THREADS : 512);
  // residency target: 4 CTAs of 256 threads (64 regs) for small N, else 1-2
  // (A/B on B200: best of {3,4} x {2,3} for T = 256; 2 for T = 512; T = 1024
  // must keep 64 registers)
  static constexpr int MINB = LOGN <= 8 ? (BN_NTT_SMALL_THREADS / T > 1 ? BN_NTT_SMALL_THREADS / T : 1)
                                        : (T <= 256 ? (MT / T > 1 ? MT / T : 1) : (T == 512 ? 2 : 1));
};

// pass P covers forward stages [S0, S1); its 16 register elements are the
// indices whose bits [LO, LO+4) vary (all other bits come from the thread id).
template <int LOGN, int P, int RB = 4>
struct PassCfgR {
  static constexpr int S0 = RB * P;
  static constexpr int S1 = (RB * P + RB < LOGN) ? RB * P + RB : LOGN;
  static constexpr int LO = (LOGN - RB * (P + 1)) > 0 ? LOGN - RB * (P + 1) : 0;
};
template <int LOGN, int P>
using PassCfg = PassCfgR<LOGN, P, 4>;

template <int LO>
BN_DEV int lay(int t, int e) {
  return (t & ((1 << LO) - 1)) | (e << LO) | ((t >> LO) << (LO + 4));
}
// Bank swizzle: XOR row bits r and r<<1 into the column (conflict
// free for every pass pattern, proven in tests/test_ntt_layout.py).
BN_DEV int swz(int u) {
  const int r = (u >> 5) & 15;
  return u ^ (r ^ (r << 1));
}

template <int TPI>
BN_DEV void bar() {
  if constexpr (TPI <= 32) __syncwarp();
  else __syncthreads();
}

// One forward register pass on NV vectors at once (NV = 2: A and B are
// transformed together — every twiddle load serves both, and the two
// independent dependency chains double the ILP at the register cost the
// held A-hat used to have).
template <int LOGN, int P, bool PADDED, int NV, int R = 16>
BN_DEV void fwd_pass(uint32_t (&x)[NV][R], int t, const uint2* __restrict__ tw, uint32_t p, uint32_t p2) {
  using PS = PassCfgR<LOGN, P, (R == 32 ? 5 : 4)>;
  const int tlow = t & ((1 << PS::LO) - 1);
#pragma unroll
  for (int s = PS::S0; s < PS::S1; s++) {
    const int b = (LOGN - 1 - s) - PS::LO;
    const uint2* Ts = tw + ((1 << LOGN) - ((1 << LOGN) >> s)) + tlow;
#pragma unroll
    for (int e = 0; e < R; e++) {
      if (e & (1 << b)) continue;
      const int el = e & ((1 << b) - 1);
      if (PS::LO == 0 && el == 0) {
        // twiddle w^0 = 1 (exponent j = tlow + el << LO = 0 for every thread):
        // no multiplication, only the lazy reductions
#pragma unroll
        for (int v = 0; v < NV; v++) {
          const uint32_t xs = x[v][e], ys = x[v][e | (1 << b)];
          x[v][e] = red2(xs + ys, p2);
          x[v][e | (1 << b)] = red2(xs - ys + p2, p2);
        }
        continue;
      }
      const uint2 w = BN_DBG_TW(Ts + (el << PS::LO));
#pragma unroll
      for (int v = 0; v < NV; v++) {
        if (PADDED && P == 0 && s == 0) {
          // zero-padded input: x[e | 8] == 0, so (x + 0, (x - 0) w)
          x[v][e | (1 << b)] = shoup(x[v][e], w.x, w.y, p);
        } else {
          gs_bfly(x[v][e], x[v][e | (1 << b)], w, p, p2);
        }
      }
    }
  }
}

template <int LOGN, int P, int R = 16>
BN_DEV void inv_pass(uint32_t (&x)[R], int t, const uint2* __restrict__ tw, uint32_t p, uint32_t p2) {
  using PS = PassCfgR<LOGN, P, (R == 32 ? 5 : 4)>;
  const int tlow = t & ((1 << PS::LO) - 1);
#pragma unroll
  for (int s = PS::S1 - 1; s >= PS::S0; s--) {
    const int b = (LOGN - 1 - s) - PS::LO;
    const uint2* Ts = tw + ((1 << LOGN) - ((1 << LOGN) >> s)) + tlow;
#pragma unroll
    for (int e = 0; e < R; e++) {
      if (e & (1 << b)) continue;
      const int el = e & ((1 << b) - 1);
      if (PS::LO == 0 && el == 0) {  // w^0 = 1
        const uint32_t u = red2(x[e], p2), v = red2(x[e | (1 << b)], p2);
        x[e] = u + v;
        x[e | (1 << b)] = u - v + p2;
        continue;
      }
      const uint2 w = BN_DBG_TW(Ts + (el << PS::LO));
      ct_bfly(x[e], x[e | (1 << b)], w, p, p2);
    }
  }
}

// Exchange-buffer addressing.  X0 = the CTA's exchange area, xo = slot * N;
// element (t, e) of a pass with low bit LO lives at CTA-wide index
// u = xo + T(t) + (e << LO), T(t) = the thread's bits outside [LO, LO+4).
//  * LOGN <= 8 (several instances per warp): additive pad u + (u >> 4) —
//    bank-conflict free for every pass pattern of these sizes
//    (tests/test_ntt_layout.py) and, being additive over the disjoint bit
//    fields of T and e, the e part folds into the LDS/STS immediate offset.
//  * LOGN >= 9: XOR swizzle swz (linear over XOR), split as
//    swz(T) ^ [e part]: the e bits above bit 4 are added (disjoint bits),
//    only the bank bits need one LOP3 per distinct constant.
template <int LOGN, int LO>
BN_DEV int xbase(int xo, int t) {
  const int T = xo + ((t & ((1 << LO) - 1)) | ((t >> LO) << (LO + 4)));
  if constexpr (LOGN <= 8) return T + (T >> 4);
  else return swz(T);
}
template <int LOGN, int LO>
BN_DEV int xaddr(int base, int e) {
  const int E = e << LO;
  if constexpr (LOGN <= 8) {
    return base + E + (E >> 4);
  } else {
    const int hE = swz(E) ^ E;  // bank-bit part of the swizzle of E
    if constexpr (LO >= 5) return (base ^ hE) + E;
    else return (base ^ ((E & 31) ^ hE)) + (E & ~31);
  }
}

// Exchange NV register vectors between pass layouts; vector v uses the plane
// X0 + v * PLANE (PLANE = the CTA's exchange-area size XW).
template <int LOGN, int LO_FROM, int LO_TO, int TPI, int NV, int PLANE>
BN_DEV void xchg(uint32_t (&x)[NV][16], uint32_t* X0, int xo, int t) {
  bar<TPI>();  // previous readers of X are done
  const int bw = xbase<LOGN, LO_FROM>(xo, t);
#pragma unroll
  for (int v = 0; v < NV; v++)
#pragma unroll
    for (int e = 0; e < 16; e++) X0[v * PLANE + xaddr<LOGN, LO_FROM>(bw, e)] = x[v][e];
  bar<TPI>();
  const int br = xbase<LOGN, LO_TO>(xo, t);
#pragma unroll
  for (int v = 0; v < NV; v++)
#pragma unroll
    for (int e = 0; e < 16; e++) x[v][e] = X0[v * PLANE + xaddr<LOGN, LO_TO>(br, e)];
}

template <int LOGN, bool PADDED, int NV, int TTA = BN_NTT_TT>
BN_DEV void fwd_all(uint32_t (&x)[NV][16], uint32_t* X0, int xo, int t, const uint2* tw, uint32_t p,
                    uint32_t p2) {
  using C = NttCfg<LOGN, TTA>;
  constexpr int PL = C::XW;
  fwd_pass<LOGN, 0, PADDED, NV>(x, t, tw, p, p2);
  if constexpr (C::NP > 1) {
    xchg<LOGN, PassCfg<LOGN, 0>::LO, PassCfg<LOGN, 1>::LO, C::TPI, NV, PL>(x, X0, xo, t);
    fwd_pass<LOGN, 1, PADDED, NV>(x, t, tw, p, p2);
  }
  if constexpr (C::NP > 2) {
    xchg<LOGN, PassCfg<LOGN, 1>::LO, PassCfg<LOGN, 2>::LO, C::TPI, NV, PL>(x, X0, xo, t);
    fwd_pass<LOGN, 2, PADDED, NV>(x, t, tw, p, p2);
  }
  if constexpr (C::NP > 3) {
    xchg<LOGN, PassCfg<LOGN, 2>::LO, PassCfg<LOGN, 3>::LO, C::TPI, NV, PL>(x, X0, xo, t);
    fwd_pass<LOGN, 3, PADDED, NV>(x, t, tw, p, p2);
  }
  static_assert(C::NP <= 4, "LOGN <= 16");
}

template <int LOGN, int TTA = BN_NTT_TT>
BN_DEV void inv_all(uint32_t (&x1)[16], uint32_t* X0, int xo, int t, const uint2* tw, uint32_t p, uint32_t p2) {
  using C = NttCfg<LOGN, TTA>;
  constexpr int PL = C::XW;
  uint32_t(&x)[1][16] = reinterpret_cast<uint32_t(&)[1][16]>(x1);
  if constexpr (C::NP > 3) {
    inv_pass<LOGN, 3>(x1, t, tw, p, p2);
    xchg<LOGN, PassCfg<LOGN, 3>::LO, PassCfg<LOGN, 2>::LO, C::TPI, 1, PL>(x, X0, xo, t);
  }
  if constexpr (C::NP > 2) {
    inv_pass<LOGN, 2>(x1, t, tw, p, p2);
    xchg<LOGN, PassCfg<LOGN, 2>::LO, PassCfg<LOGN, 1>::LO, C::TPI, 1, PL>(x, X0, xo, t);
  }
  if constexpr (C::NP > 1) {
    inv_pass<LOGN, 1>(x1, t, tw, p, p2);
    xchg<LOGN, PassCfg<LOGN, 1>::LO, PassCfg<LOGN, 0>::LO, C::TPI, 1, PL>(x, X0, xo, t);
  }
  inv_pass<LOGN, 0>(x1, t, tw, p, p2);
}

// 3-word accumulate (a0, a1, a2) += (c0, c1, c2)
BN_DEV void add3(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t c0, uint32_t c1, uint32_t c2) {
  asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
      : "+r"(a0), "+r"(a1), "+r"(a2)
      : "r"(c0), "r"(c1), "r"(c2));
}

// ------------------------------------------------------------ epilogue layout
// Residue arrays are written in a pass layout (consecutive threads ->
// consecutive words) and read back as Q consecutive words per thread with
// 128-bit accesses; the L / H arrays are written and read Q words per
// thread.  Row-major, the 8 threads of a quarter-warp access 16-byte chunks
// 4Q bytes apart: a 2-way (Q = 8) or 4-way (Q = 16) bank conflict (ncu r02:
// 14% of the shared wavefronts at 4K, 22% at 128K / 256K).  The Q = 16
// kernels (32-element, wide, cluster32) use the cswz<16> layout
// (bn_common.cuh): A/B on B200 (ms per paper batch) wide 4K 3.42 -> 3.23,
// 16K 4.52 -> 4.35, 128K 7.34 -> 7.11; mul_ntt 256K 6.53 -> 6.45.  The
// Q = 8 16-element kernels keep the plain layout (S = false): there the
// issue slots are the binding limit and the swizzle's address arithmetic
// cost more than the 2-way conflicts (4K 2.873 -> 2.904, 16K 3.81 -> 3.86).
// NW words at logical index k0 (a multiple of 4) of a cswz<Q> array
template <int Q, int NW, bool S = true>
BN_DEV void lds_swz(uint32_t (&r)[NW], const uint32_t* base, int k0) {
#pragma unroll
  for (int v = 0; v < NW / 4; v++) {
    const uint4 x = *reinterpret_cast<const uint4*>(base + cswz<Q, S>(k0 + 4 * v));
    r[4 * v + 0] = x.x; r[4 * v + 1] = x.y; r[4 * v + 2] = x.z; r[4 * v + 3] = x.w;
  }
}
template <int Q, int NW, bool S = true>
BN_DEV void sts_swz(uint32_t* base, int k0, const uint32_t (&r)[NW]) {
#pragma unroll
  for (int v = 0; v < NW / 4; v++)
    *reinterpret_cast<uint4*>(base + cswz<Q, S>(k0 + 4 * v)) =
        make_uint4(r[4 * v + 0], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
}

// N-5 / N-6: Garner CRT (reading R10) of the Q consecutive coefficients
// k0 .. k0+Q-1, read from the three residue arrays Res + j RS (cswz<Q>
// layout), with the inverse-transform scale 2^32 N^-1 folded into the
// constants, then aggregated: S = sum_q c_{k0+q} 2^(32 q) -> lows[q] = limb q
// of S, (h0, h1) = the two words above it (S >> 32Q < 2^46).
//   r0 = y0 K0 mod p0
//   t1 = (y1 K1 - r0) p0^-1 mod p1
//   t2 = (y2 K2 - r0 - p0 t1) (p0 p1)^-1 mod p2
//   c  = r0 + p0 t1 + p0 p1 t2  (< 2^90; c < m (2^32-1)^2 exactly)
// G: the residues are in global memory (the Poly kernel's workspace, written
// in this kernel: coherent ld.global.cg, row-major) instead of shared memory.
template <int Q, bool S, bool G = false>
BN_DEV void crt_aggregate(const uint32_t* Res, int RS, int k0, const CrtConst& k, uint32_t (&lows)[Q],
                          uint32_t& h0, uint32_t& h1) {
  const uint32_t p0 = c_pc[0].p, p1 = c_pc[1].p, p2 = c_pc[2].p;
  uint32_t a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
  for (int h = 0; h < Q / 8; h++) {
    uint32_t y0[8], y1[8], y2[8];
    if constexpr (G) {
      ldcg_limbs<8>(y0, Res + 0 * RS + k0 + 8 * h);
      ldcg_limbs<8>(y1, Res + 1 * RS + k0 + 8 * h);
      ldcg_limbs<8>(y2, Res + 2 * RS + k0 + 8 * h);
    } else {
      lds_swz<Q, 8, S>(y0, Res + 0 * RS, k0 + 8 * h);
      lds_swz<Q, 8, S>(y1, Res + 1 * RS, k0 + 8 * h);
      lds_swz<Q, 8, S>(y2, Res + 2 * RS, k0 + 8 * h);
    }
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const uint32_t r0 = red2(shoup(y0[q], k.k0, k.k0_sh, p0), p0);
      const uint32_t u = shoup(y1[q], k.k1i, k.k1i_sh, p1);
      const uint32_t v = shoup(r0, k.i01, k.i01_sh, p1);
      const uint32_t t1 = red2(red2(u + 2 * p1 - v, 2 * p1), p1);
      const uint32_t a2v = shoup(y2[q], k.k2i, k.k2i_sh, p2);
      const uint32_t b2v = shoup(r0, k.i012, k.i012_sh, p2);
      const uint32_t c2v = shoup(t1, k.p0i012, k.p0i012_sh, p2);
      const uint32_t d = red2(b2v + c2v, 2 * p2);
      const uint32_t t2 = red2(red2(a2v + 2 * p2 - d, 2 * p2), p2);
      const uint64_t v64 = (uint64_t)p0 * t1 + r0;
      const uint64_t w = (uint64_t)k.p01_lo * t2 + v64;
      const uint64_t hh = (uint64_t)k.p01_hi * t2 + (w >> 32);
      add3(a0, a1, a2, (uint32_t)w, (uint32_t)hh, (uint32_t)(hh >> 32));
      lows[8 * h + q] = a0;
      a0 = a1;
      a1 = a2;
      a2 = 0;
    }
  }
  h0 = a0;
  h1 = a1;
}

// Publish (reading R8, as the classical kernel): L[k0 .. k0+Q) = lows,
// H[k0+Q] = h0, H[k0+Q+1] = h1, H[k0+Q+2 .. k0+2Q) = 0; the top chunk
// (k0 + Q == M) zeroes H[0 .. Q) instead (positions >= M are dropped).
// L and H are cswz<Q> arrays of M words.
template <int Q, bool S>
BN_DEV void publish_lh(uint32_t* L, uint32_t* H, int k0, int M, const uint32_t (&lows)[Q], uint32_t h0,
                       uint32_t h1) {
  uint32_t hs[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) hs[q] = q == 0 ? h0 : (q == 1 ? h1 : 0u);
  sts_swz<Q, Q, S>(L, k0, lows);
  if (k0 + Q < M) {
    sts_swz<Q, Q, S>(H, k0 + Q, hs);
  } else {
#pragma unroll
    for (int q = 0; q < Q; q++) hs[q] = 0;
    sts_swz<Q, Q, S>(H, 0, hs);
  }
}

// ------------------------------------------------------------ one product
// The pieces of one NTT product for one instance slot of the 16-element
// layout, used by the fused Poly kernel:
//  * ntt_residues: per prime N-1..N-4 — reduce, forward transform(s),
//    pointwise product, inverse — leaving the raw inverse outputs of
//    coefficients 0..M-1 in Res[j M + k] (three arrays of M words);
//  * ntt_epilogue: N-5..N-7 — Garner CRT + aggregate + L / H publish (into
//    the slot's exchange region X), resolve R = L + H by the scan-add and,
//    when ADD, a second scan-add of the addend (the Poly additions fused into
//    the product's epilogue), then the store.
// SQ: x == y, one forward transform serves both operands (x-hat * x-hat).
// XWS / AWS / OWS: operand / addend / destination in the in-kernel workspace
// (coherent ld.global.cg, write-back stores) instead of HBM (ld.global.nc,
// streaming stores).
template <int LOGN, bool SQ, bool XWS, int TTA>
BN_DEV void ntt_residues(uint32_t* sm, int slot, int t, const uint32_t* xi, const uint32_t* yi, uint32_t* Res,
                         bool valid, const uint2* __restrict__ tw) {
  using C = NttCfg<LOGN, TTA>;
  constexpr int N = C::N, M = C::M;
  constexpr int NV = SQ ? 1 : 2;
#pragma unroll 1
  for (int j = 0; j < kNumPrimes; j++) {
    const uint32_t p = c_pc[j].p, p2 = c_pc[j].p2, pinv = c_pc[j].pinv;
    const uint2* twf = tw + (2 * j + 0) * (N - 1);
    const uint2* twi = tw + (2 * j + 1) * (N - 1);
    uint32_t xab[NV][16];
    // N-1: reduce the limbs mod p into pass-0 layout (index t + e N/16),
    // upper half is the zero padding (reading R11)
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const uint32_t* px = xi + t + e * (N / 16);
      const uint32_t va = valid ? (XWS ? __ldcg(px) : __ldg(px)) : 0u;
      // a_i < 2^32 < 6p: two conditional subtractions of 2p -> [0, 2p)
      xab[0][e] = red2(red2(va, p2), p2);
      if constexpr (!SQ) {
        const uint32_t* py = yi + t + e * (N / 16);
        const uint32_t vb = valid ? (XWS ? __ldcg(py) : __ldg(py)) : 0u;
        xab[NV - 1][e] = red2(red2(vb, p2), p2);
      }
    }
#pragma unroll
    for (int e = 8; e < 16; e++) {
#pragma unroll
      for (int v = 0; v < NV; v++) xab[v][e] = 0u;
    }
    // N-2: forward transforms of x and y together (one when squaring)
    fwd_all<LOGN, true, NV, TTA>(xab, sm, slot * N, t, twf, p, p2);
    // N-3: pointwise product (same register layout for both transforms)
    uint32_t x[16];
#pragma unroll
    for (int e = 0; e < 16; e++) x[e] = mont(xab[0][e], xab[NV - 1][e], p, pinv);
    // N-4: inverse transform -> pass-0 layout, natural order
    inv_all<LOGN, TTA>(x, sm, slot * N, t, twi, p, p2);
    // keep coefficients 0..M-1 (truncated product): e < 8
#pragma unroll
    for (int e = 0; e < 8; e++) Res[j * M + t + e * (N / 16)] = x[e];
  }
}

template <int LOGN, bool ADD, bool AWS, bool OWS, int TTA>
BN_DEV void ntt_epilogue(uint32_t* X, const uint32_t* Res, uint32_t* agg, int t, bool valid, const uint32_t* addi,
                         uint32_t* dsti) {
  using C = NttCfg<LOGN, TTA>;
  constexpr int M = C::M, TPI = C::TPI;
  bar<TPI>();  // residues complete; X dead (its last readers were the final exchange)
  // N-5 / N-6: Garner CRT of 8 consecutive coefficients, aggregate, publish
  {
    uint32_t lows[8], h0, h1;
    crt_aggregate<8, false>(Res, M, 8 * t, c_crt[LOGN], lows, h0, h1);
    publish_lh<8, false>(X, X + M, 8 * t, M, lows, h0, h1);
  }
  bar<TPI>();
  // N-7: R = L + H (+ addend), store
  {
    uint32_t xl[8], yh[8], r[8];
    lds_swz<8, 8, false>(xl, X, 8 * t);
    lds_swz<8, 8, false>(yh, X + M, 8 * t);
    add_regs<8, TPI>(xl, yh, r, valid, agg);
    if constexpr (ADD) {
      uint32_t ad[8], r2[8];
      if (valid) load_any<AWS, 8>(ad, addi + 8 * t);
      else {
#pragma unroll
        for (int q = 0; q < 8; q++) ad[q] = 0;
      }
      if constexpr (TPI > 32) __syncthreads();  // agg reuse
      add_regs<8, TPI>(r, ad, r2, valid, agg);
      if (valid) store_any<OWS, 8>(dsti + 8 * t, r2);
    } else {
      if (valid) store_any<OWS, 8>(dsti + 8 * t, r);
    }
  }
  __syncthreads();  // X / Res / agg reused next; dst visible to the CTA
}

// Poly's first level, transform-shared: per prime, the forward transforms
// A-hat, B-hat are computed once (together), then the three pointwise
// products A-hat^2, B-hat^2, A-hat B-hat are inverse-transformed one after
// the other into Res9[(3 P + j) M + k] (P = 0: a*a, 1: b*b, 2: a*b).
// A-hat stays in registers; B-hat is parked in the slot's plane-1 region,
// which the one-vector inverse exchanges never touch (thread-private slots
// [e TPI + t]: only the owner reads them back, no barrier needed).
template <int LOGN, int TTA>
BN_DEV void ntt_residues3(uint32_t* sm, int slot, int t, const uint32_t* ai, const uint32_t* bi, uint32_t* Res9,
                          bool valid, const uint2* __restrict__ tw) {
  using C = NttCfg<LOGN, TTA>;
  constexpr int N = C::N, M = C::M, TPI = C::TPI;
  uint32_t* Bp = sm + C::XW + slot * (C::XW / C::IPB);  // plane 1 of this slot
#pragma unroll 1
  for (int j = 0; j < kNumPrimes; j++) {
    const uint32_t p = c_pc[j].p, p2 = c_pc[j].p2, pinv = c_pc[j].pinv;
    const uint2* twf = tw + (2 * j + 0) * (N - 1);
    const uint2* twi = tw + (2 * j + 1) * (N - 1);
    uint32_t xab[2][16];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const uint32_t va = valid ? __ldg(ai + t + e * (N / 16)) : 0u;
      const uint32_t vb = valid ? __ldg(bi + t + e * (N / 16)) : 0u;
      xab[0][e] = red2(red2(va, p2), p2);
      xab[1][e] = red2(red2(vb, p2), p2);
    }
#pragma unroll
    for (int e = 8; e < 16; e++) xab[0][e] = xab[1][e] = 0u;
    fwd_all<LOGN, true, 2, TTA>(xab, sm, slot * N, t, twf, p, p2);
    bar<TPI>();  // every read of plane 1 by the last forward exchange is done
#pragma unroll
    for (int e = 0; e < 16; e++) Bp[e * TPI + t] = xab[1][e];
    uint32_t(&ah)[16] = xab[0];
#pragma unroll 1
    for (int P = 0; P < 3; P++) {
      uint32_t x[16];
#pragma unroll
      for (int e = 0; e < 16; e++) {
        const uint32_t bh = P == 0 ? 0u : Bp[e * TPI + t];
        x[e] = mont(P == 1 ? bh : ah[e], P == 0 ? ah[e] : bh, p, pinv);
      }
      inv_all<LOGN, TTA>(x, sm, slot * N, t, twi, p, p2);
#pragma unroll
      for (int e = 0; e < 8; e++) Res9[(3 * P + j) * M + t + e * (N / 16)] = x[e];
    }
  }
}

// ------------------------------------------------------------ the kernels
// The 1-Mul kernel keeps its body inline instead of calling ntt_product:
// routed through the helper, ptxas allocates registers differently and the
// 1024-bit instance runs 6-9% slower (A/B on one B200, scripts/ab.sh).
template <int LOGN>
__global__ void __launch_bounds__(NttCfg<LOGN>::T, NttCfg<LOGN>::MINB)
    mul_ntt_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                   const uint2* __restrict__ tw) {
  using C = NttCfg<LOGN>;
  constexpr int N = C::N, M = C::M, TPI = C::TPI;
  extern __shared__ __align__(16) uint32_t sm[];
  const int slot = threadIdx.x / TPI;
  const int t = threadIdx.x % TPI;
  // this slot's own (padded) exchange region, reused for L | H after the
  // transforms: it must not reach into another slot's region, because slots
  // in different warps only synchronise at CTA barriers
  uint32_t* X = sm + slot * (C::XW / C::IPB);
  // raw inverse outputs per prime; per-slot stride padded by 16 words so the two
  // instances sharing a warp (TPI = 16) write different banks
  constexpr int RS = 3 * M + (C::TPI < 32 ? 16 : 0);
  uint32_t* Res = sm + 2 * C::XW + slot * RS;
  uint32_t* agg = sm + 2 * C::XW + C::IPB * RS;

  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  for (uint64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const uint64_t inst = grp * C::IPB + slot;
    const bool valid = inst < n_inst;
    const uint32_t* ai = a + (valid ? inst : 0) * M;
    const uint32_t* bi = b + (valid ? inst : 0) * M;

#pragma unroll 1
    for (int j = 0; j < kNumPrimes; j++) {
      const uint32_t p = c_pc[j].p, p2 = c_pc[j].p2, pinv = c_pc[j].pinv;
      const uint2* twf = tw + (2 * j + 0) * (N - 1);
      const uint2* twi = tw + (2 * j + 1) * (N - 1);
      uint32_t xab[2][16];
      // N-1: reduce the limbs mod p into pass-0 layout (index t + e N/16),
      // upper half is the zero padding (reading R11)
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const uint32_t va = valid ? __ldg(ai + t + e * (N / 16)) : 0u;
        const uint32_t vb = valid ? __ldg(bi + t + e * (N / 16)) : 0u;
        // a_i < 2^32 < 6p: two conditional subtractions of 2p -> [0, 2p)
        xab[0][e] = red2(red2(va, p2), p2);
        xab[1][e] = red2(red2(vb, p2), p2);
      }
#pragma unroll
      for (int e = 8; e < 16; e++) xab[0][e] = xab[1][e] = 0u;
      // N-2: forward transforms of A and B together
      fwd_all<LOGN, true, 2>(xab, sm, slot * N, t, twf, p, p2);
      // N-3: pointwise product (same register layout for A-hat and B-hat)
      uint32_t x[16];
#pragma unroll
      for (int e = 0; e < 16; e++) x[e] = mont(xab[0][e], xab[1][e], p, pinv);
      // N-4: inverse transform -> pass-0 layout, natural order
      inv_all<LOGN>(x, sm, slot * N, t, twi, p, p2);
      // keep coefficients 0..M-1 (truncated product): e < 8
#pragma unroll
      for (int e = 0; e < 8; e++) Res[j * M + cswz<8, false>(t + e * (N / 16))] = x[e];
    }
    bar<TPI>();

    // N-5 / N-6: Garner CRT of 8 consecutive coefficients, aggregate, publish
    // (X is dead: the last exchange read it before inv_pass<0>, then bar)
    {
      uint32_t lows[8], h0, h1;
      crt_aggregate<8, false>(Res, M, 8 * t, c_crt[LOGN], lows, h0, h1);
      publish_lh<8, false>(X, X + M, 8 * t, M, lows, h0, h1);
    }
    bar<TPI>();
    // N-7: R = L + H, store
    {
      uint32_t xl[8], yh[8], r[8];
      lds_swz<8, 8, false>(xl, X, 8 * t);
      lds_swz<8, 8, false>(yh, X + M, 8 * t);
      add_regs<8, TPI>(xl, yh, r, valid, agg);
      if (valid) store_limbs<8>(out + inst * M + 8 * t, r);
    }
    __syncthreads();  // X / Res / agg reused by the next group
  }
}

// Poly (Table 2 caption): (a*a + b) * (b*b + b) + a*b
// mod 2^bits in ONE kernel — four NTT products with the three additions
// fused into their epilogues (block-level fusion).  The three first-level
// products share their forward transforms (ntt_residues3): per prime
// 2 forward + 3 inverse transforms, then t1 * t2 costs 2 + 1, so a Poly is
// 8 transforms per prime (four independent products: 12; squaring reuse
// alone: 10).  The residues of the first level (9 M words per instance)
// stay in shared memory; t1 = a^2 + b, t2 = b^2 + b, t3 = a b go to this
// CTA's private workspace slice (L2-resident, rewritten by the same CTA group
// after group) and are read back coherently by the last product.
template <int LOGN>
struct PolyNttCfg {
  using B = NttCfg<LOGN, kPolyNttTT>;
  static constexpr int RS = 9 * B::M + (B::TPI < 32 ? 16 : 0);  // per slot: [3 P + j][M]
  static constexpr int SMEM_WORDS = 2 * B::XW + B::IPB * RS + B::T / 32;
  // residency the shared memory allows (227 KiB per SM): never ask ptxas to
  // cap registers for CTAs that could not be co-resident anyway
  static constexpr int BY_SMEM = (227 * 1024) / (SMEM_WORDS * 4);
  static constexpr int MINB = BY_SMEM < 1 ? 1 : (BY_SMEM < B::MINB ? BY_SMEM : B::MINB);
};

template <int LOGN>
__global__ void __launch_bounds__(NttCfg<LOGN, kPolyNttTT>::T, PolyNttCfg<LOGN>::MINB)
    poly_ntt_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                    const uint2* __restrict__ tw, uint32_t* ws) {
  using C = NttCfg<LOGN, kPolyNttTT>;
  using PC = PolyNttCfg<LOGN>;
  constexpr int M = C::M;
  extern __shared__ __align__(16) uint32_t sm[];
  const int slot = threadIdx.x / C::TPI;
  const int t = threadIdx.x % C::TPI;
  uint32_t* X = sm + slot * (C::XW / C::IPB);
  uint32_t* Res9 = sm + 2 * C::XW + slot * PC::RS;
  uint32_t* agg = sm + 2 * C::XW + C::IPB * PC::RS;
  uint32_t* t1 = ws + ((uint64_t)blockIdx.x * C::IPB + slot) * 3 * M;
  uint32_t* t2 = t1 + M;
  uint32_t* t3 = t2 + M;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  for (uint64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const uint64_t inst = grp * C::IPB + slot;
    const bool valid = inst < n_inst;
    const uint64_t io = (valid ? inst : 0) * M;
    const uint32_t* ai = a + io;
    const uint32_t* bi = b + io;
    constexpr int TT = kPolyNttTT;
    ntt_residues3<LOGN, TT>(sm, slot, t, ai, bi, Res9, valid, tw);
    //               ADD    AWS    OWS
    ntt_epilogue<LOGN, true, false, true, TT>(X, Res9 + 0 * M, agg, t, valid, bi, t1);   // a^2 + b
    ntt_epilogue<LOGN, true, false, true, TT>(X, Res9 + 3 * M, agg, t, valid, bi, t2);   // b^2 + b
    ntt_epilogue<LOGN, false, false, true, TT>(X, Res9 + 6 * M, agg, t, valid, nullptr, t3);  // a b
    //                SQ     XWS
    ntt_residues<LOGN, false, true, TT>(sm, slot, t, t1, t2, Res9, valid, tw);
    ntt_epilogue<LOGN, true, true, false, TT>(X, Res9, agg, t, valid, t3, out + io);  // t1 t2 + t3
  }
}

// ------------------------------------------------------------ 32 elements per thread
// N = 2^13, 2^14 (128K / 256K bits): T = N / 32 threads (256 / 512) each
// holding R = 32 register elements, 5 stages per register pass, so a
// transform is 3 passes / 2 exchanges instead of 4 / 3, and the thread count
// drops to where up to 128 registers are available (no spills; the 16-element
// kernel at 1024 threads is capped at 64).  Exchange addresses: element
// (t, e) of a pass with low bit LO lives at u = lay(t, e) with 5 register
// bits, swizzled u ^ ((u >> 5) & 31) — for a warp (32 consecutive t, fixed
// e) the 5 bank bits are a bijection of t's low 5 bits for every LO, so
// every exchange access is conflict free.  Epilogue: 16 consecutive
// coefficients per thread (M / T = 16), resolved 16 limbs per thread.
template <int LOGN>
struct NttR32Cfg {
  static constexpr int N = 1 << LOGN, M = N / 2, R = 32, RB = 5;
  static constexpr int T = N / R;
  static constexpr int SMEM_WORDS = 2 * N + 3 * M + T / 32;
  static constexpr int MINB = T <= 256 ? 2 : 1;  // <= 128 registers
  static_assert((LOGN + RB - 1) / RB == 3, "three register passes");
};

BN_DEV int swz5(int u) { return u ^ ((u >> 5) & 31); }
template <int LO>
BN_DEV int lay32(int t, int e) {
  return (t & ((1 << LO) - 1)) | (e << LO) | ((t >> LO) << (LO + 5));
}

template <int LO_FROM, int LO_TO, int NV, int PLANE>
BN_DEV void xchg32(uint32_t (&x)[NV][32], uint32_t* X0, int t) {
  __syncthreads();  // previous readers of the planes are done
  const int bw = swz5(lay32<LO_FROM>(t, 0));
#pragma unroll
  for (int v = 0; v < NV; v++)
#pragma unroll
    for (int e = 0; e < 32; e++) X0[v * PLANE + (bw ^ swz5(e << LO_FROM))] = x[v][e];
  __syncthreads();
  const int br = swz5(lay32<LO_TO>(t, 0));
#pragma unroll
  for (int v = 0; v < NV; v++)
#pragma unroll
    for (int e = 0; e < 32; e++) x[v][e] = X0[v * PLANE + (br ^ swz5(e << LO_TO))];
}

template <int LOGN>
__global__ void __launch_bounds__(NttR32Cfg<LOGN>::T, NttR32Cfg<LOGN>::MINB)
    mul_ntt_r32_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                       const uint2* __restrict__ tw) {
  using C = NttR32Cfg<LOGN>;
  constexpr int N = C::N, M = C::M, T = C::T;
  constexpr int L0 = PassCfgR<LOGN, 0, 5>::LO, L1 = PassCfgR<LOGN, 1, 5>::LO, L2 = PassCfgR<LOGN, 2, 5>::LO;
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* X = sm;              // plane 0 | plane 1 (N words each)
  uint32_t* Res = sm + 2 * N;    // 3 M residues
  uint32_t* agg = Res + 3 * M;   // T / 32
  const int t = threadIdx.x;
  // Raw limbs of the next (prime, instance) step, in pass-0 layout (index
  // t + e N/32).  With one 512-thread CTA per SM nothing else hides a load,
  // so the limbs for prime j + 1 (or the next instance's prime 0) are issued
  // before prime j's inverse transform and consumed after it.
  constexpr bool PF = LOGN <= BN_NTT_R32_PREFETCH_MAXLOG;
  uint32_t ra[16], rb[16];
  auto fetch = [&](uint64_t i) {
    const uint32_t* ai = a + i * M + t;
    const uint32_t* bi = b + i * M + t;
#pragma unroll
    for (int e = 0; e < 16; e++) {
      ra[e] = __ldg(ai + e * (N / 32));
      rb[e] = __ldg(bi + e * (N / 32));
    }
  };
  if (PF && blockIdx.x < n_inst) fetch(blockIdx.x);
  for (uint64_t inst = blockIdx.x; inst < n_inst; inst += gridDim.x) {
#pragma unroll 1
    for (int j = 0; j < kNumPrimes; j++) {
      const uint32_t p = c_pc[j].p, p2 = c_pc[j].p2, pinv = c_pc[j].pinv;
      const uint2* twf = tw + (2 * j + 0) * (N - 1);
      const uint2* twi = tw + (2 * j + 1) * (N - 1);
      uint32_t xab[2][32];
      if constexpr (!PF) fetch(inst);
      // N-1: limbs mod p in pass-0 layout (index t + e N/32), top half zero
#pragma unroll
      for (int e = 0; e < 16; e++) {
        xab[0][e] = red2(red2(ra[e], p2), p2);
        xab[1][e] = red2(red2(rb[e], p2), p2);
      }
#pragma unroll
      for (int e = 16; e < 32; e++) xab[0][e] = xab[1][e] = 0u;
      // N-2: forward DIF, 3 passes
      fwd_pass<LOGN, 0, true, 2, 32>(xab, t, twf, p, p2);
      xchg32<L0, L1, 2, N>(xab, X, t);
      fwd_pass<LOGN, 1, true, 2, 32>(xab, t, twf, p, p2);
      xchg32<L1, L2, 2, N>(xab, X, t);
      fwd_pass<LOGN, 2, true, 2, 32>(xab, t, twf, p, p2);
      // N-3: pointwise
      uint32_t x[1][32];
#pragma unroll
      for (int e = 0; e < 32; e++) x[0][e] = mont(xab[0][e], xab[1][e], p, pinv);
      if constexpr (PF) {
        const uint64_t nxt = j + 1 < kNumPrimes ? inst : inst + gridDim.x;
        if (nxt < n_inst) fetch(nxt);
      }
      // N-4: inverse DIT, 3 passes back to the pass-0 layout
      inv_pass<LOGN, 2, 32>(x[0], t, twi, p, p2);
      xchg32<L2, L1, 1, N>(x, X, t);
      inv_pass<LOGN, 1, 32>(x[0], t, twi, p, p2);
      xchg32<L1, L0, 1, N>(x, X, t);
      inv_pass<LOGN, 0, 32>(x[0], t, twi, p, p2);
#pragma unroll
      for (int e = 0; e < 16; e++) Res[j * M + cswz<16>(t + e * (N / 32))] = x[0][e];
    }
    __syncthreads();

    // N-5 / N-6: Garner CRT of 16 consecutive coefficients, aggregate, publish
    {
      uint32_t lows[16], h0, h1;
      crt_aggregate<16, true>(Res, M, 16 * t, c_crt[LOGN], lows, h0, h1);
      publish_lh<16, true>(X, X + N, 16 * t, M, lows, h0, h1);
    }
    __syncthreads();
    {
      uint32_t xl[16], yh[16], r[16];
      lds_swz<16, 16>(xl, X, 16 * t);
      lds_swz<16, 16>(yh, X + N, 16 * t);
      add_regs<16, T>(xl, yh, r, true, agg);
      store_limbs<16>(out + inst * M + 16 * t, r);
    }
    __syncthreads();
  }
}

template <int LOGN>
static cudaError_t launch_ntt_r32_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                    const NttTables& tb, cudaStream_t st, int n_sm) {
  using C = NttR32Cfg<LOGN>;
#ifdef BN_DBG_R32_SMEM_KB  // timing experiment: pad the shared memory request (residency)
  constexpr size_t need = C::SMEM_WORDS * sizeof(uint32_t);
  constexpr size_t smem = need > (size_t)BN_DBG_R32_SMEM_KB * 1024 ? need : (size_t)BN_DBG_R32_SMEM_KB * 1024;
#else
  constexpr size_t smem = C::SMEM_WORDS * sizeof(uint32_t);
#endif
  static LaunchCache cache;
  int per_sm = 0;
  cudaError_t e = resident_ctas(cache, mul_ntt_r32_kernel<LOGN>, C::T, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t cap = (uint64_t)n_sm * per_sm;
  const unsigned grid = cap_grid((unsigned)(n_inst < cap ? n_inst : cap));
  mul_ntt_r32_kernel<LOGN><<<grid, C::T, smem, st>>>(out, a, b, n_inst, tb.tw);
  return cudaGetLastError();
}

// Poly at N = 2^13, 2^14 (128K / 256K bits) on the 32-element layout: the
// 16-element kernel would need 1024-thread CTAs capped at 64 registers
// (spills) and, at 2^14, more shared memory than a CTA has for the 9 M
// first-level residues.  Same transform sharing as poly_ntt_kernel
// (8 transforms per prime); the first-level residues go to the CTA's
// workspace slice in global memory (L2-resident; written coalesced in the
// pass-0 layout, read back 16 consecutive words per thread), the last
// product's residues stay in shared memory as in the 1-Mul kernel.
// Workspace per resident CTA: G9 (9 M words) | t1 | t2 | t3 (M words each).
template <int LOGN>
struct PolyR32Cfg {
  using B = NttR32Cfg<LOGN>;
  static constexpr int WS_WORDS = 12 * B::M;
};

template <int LOGN>
BN_DEV void r32_fwd(uint32_t (&xab)[2][32], uint32_t* X, int t, const uint2* twf, uint32_t p, uint32_t p2) {
  constexpr int N = 1 << LOGN;
  constexpr int L0 = PassCfgR<LOGN, 0, 5>::LO, L1 = PassCfgR<LOGN, 1, 5>::LO, L2 = PassCfgR<LOGN, 2, 5>::LO;
  fwd_pass<LOGN, 0, true, 2, 32>(xab, t, twf, p, p2);
  xchg32<L0, L1, 2, N>(xab, X, t);
  fwd_pass<LOGN, 1, true, 2, 32>(xab, t, twf, p, p2);
  xchg32<L1, L2, 2, N>(xab, X, t);
  fwd_pass<LOGN, 2, true, 2, 32>(xab, t, twf, p, p2);
}

template <int LOGN>
BN_DEV void r32_fwd1(uint32_t (&x)[1][32], uint32_t* X, int t, const uint2* twf, uint32_t p, uint32_t p2) {
  constexpr int N = 1 << LOGN;
  constexpr int L0 = PassCfgR<LOGN, 0, 5>::LO, L1 = PassCfgR<LOGN, 1, 5>::LO, L2 = PassCfgR<LOGN, 2, 5>::LO;
  fwd_pass<LOGN, 0, true, 1, 32>(x, t, twf, p, p2);
  xchg32<L0, L1, 1, N>(x, X, t);
  fwd_pass<LOGN, 1, true, 1, 32>(x, t, twf, p, p2);
  xchg32<L1, L2, 1, N>(x, X, t);
  fwd_pass<LOGN, 2, true, 1, 32>(x, t, twf, p, p2);
}

template <int LOGN>
BN_DEV void r32_inv(uint32_t (&x)[1][32], uint32_t* X, int t, const uint2* twi, uint32_t p, uint32_t p2) {
  constexpr int N = 1 << LOGN;
  constexpr int L0 = PassCfgR<LOGN, 0, 5>::LO, L1 = PassCfgR<LOGN, 1, 5>::LO, L2 = PassCfgR<LOGN, 2, 5>::LO;
  inv_pass<LOGN, 2, 32>(x[0], t, twi, p, p2);
  xchg32<L2, L1, 1, N>(x, X, t);
  inv_pass<LOGN, 1, 32>(x[0], t, twi, p, p2);
  xchg32<L1, L0, 1, N>(x, X, t);
  inv_pass<LOGN, 0, 32>(x[0], t, twi, p, p2);
}

// raw limbs of x, y (16 each, pass-0 layout t + e N/32) reduced mod p
template <int LOGN, bool XWS>
BN_DEV void r32_load(uint32_t (&xab)[2][32], const uint32_t* xi, const uint32_t* yi, int t, uint32_t p2) {
  constexpr int N = 1 << LOGN;
#pragma unroll
  for (int e = 0; e < 16; e++) {
    const uint32_t* px = xi + t + e * (N / 32);
    const uint32_t* py = yi + t + e * (N / 32);
    xab[0][e] = red2(red2(XWS ? __ldcg(px) : __ldg(px), p2), p2);
    xab[1][e] = red2(red2(XWS ? __ldcg(py) : __ldg(py), p2), p2);
  }
#pragma unroll
  for (int e = 16; e < 32; e++) xab[0][e] = xab[1][e] = 0u;
}

// N-5..N-7 on the 32-element layout: CRT of 16 consecutive coefficients
// (residues in shared memory, cswz<16>, or in global memory when G), L / H
// publish into the planes, resolve (+ addend), store.  Brackets itself with
// CTA barriers.
template <int LOGN, bool G, bool ADD, bool AWS, bool OWS>
BN_DEV void r32_epilogue(uint32_t* X, const uint32_t* Res, uint32_t* agg, int t, const uint32_t* addi,
                         uint32_t* dsti) {
  constexpr int N = 1 << LOGN, M = N / 2, T = N / 32;
  __syncthreads();  // residues complete (shared or global); planes dead
  {
    uint32_t lows[16], h0, h1;
    crt_aggregate<16, true, G>(Res, M, 16 * t, c_crt[LOGN], lows, h0, h1);
    publish_lh<16, true>(X, X + N, 16 * t, M, lows, h0, h1);
  }
  __syncthreads();
  {
    uint32_t xl[16], yh[16], r[16];
    lds_swz<16, 16>(xl, X, 16 * t);
    lds_swz<16, 16>(yh, X + N, 16 * t);
    add_regs<16, T>(xl, yh, r, true, agg);
    if constexpr (ADD) {
      uint32_t ad[16], r2[16];
      load_any<AWS, 16>(ad, addi + 16 * t);
      __syncthreads();  // agg reuse
      add_regs<16, T>(r, ad, r2, true, agg);
      store_any<OWS, 16>(dsti + 16 * t, r2);
    } else {
      store_any<OWS, 16>(dsti + 16 * t, r);
    }
  }
  __syncthreads();  // planes / agg reused next; dst visible to the CTA
}

template <int LOGN>
__global__ void __launch_bounds__(NttR32Cfg<LOGN>::T, NttR32Cfg<LOGN>::MINB)
    poly_ntt_r32_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                        const uint2* __restrict__ tw, uint32_t* ws) {
  using C = NttR32Cfg<LOGN>;
  constexpr int N = C::N, M = C::M;
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* X = sm;              // plane 0 | plane 1 (N words each)
  uint32_t* Park = sm + 2 * N;   // A-hat parked here (the 1-Mul kernel's residue area)
  uint32_t* agg = Park + 3 * M;  // T / 32
  const int t = threadIdx.x;
  uint32_t* G9 = ws + (uint64_t)blockIdx.x * PolyR32Cfg<LOGN>::WS_WORDS;  // [3 P + j][M]
  uint32_t* t1 = G9 + 9 * M;
  uint32_t* t2 = t1 + M;
  uint32_t* t3 = t2 + M;
  for (uint64_t inst = blockIdx.x; inst < n_inst; inst += gridDim.x) {
    // Two phases through ONE copy of the transform code (phase 0: the three
    // first-level products of a, b; phase 1: t1 * t2), so ptxas allocates
    // registers for a single transform body (two inlined bodies spilled
    // 430-560 bytes per thread).  Every product's residues go to the
    // workspace (G9), every epilogue reads them from there.
#pragma unroll 1
    for (int phase = 0; phase < 2; phase++) {
      const uint32_t* xi = phase ? t1 : a + inst * M;
      const uint32_t* yi = phase ? t2 : b + inst * M;
      const int P0 = phase ? 2 : 0;  // phase 1: the single product t1 * t2, into G9 slot 2
#pragma unroll 1
      for (int j = 0; j < kNumPrimes; j++) {
        const uint32_t p = c_pc[j].p, p2 = c_pc[j].p2, pinv = c_pc[j].pinv;
        const uint2* twf = tw + (2 * j + 0) * (N - 1);
        const uint2* twi = tw + (2 * j + 1) * (N - 1);
        {
          uint32_t xab[2][32];
          r32_load<LOGN, true>(xab, xi, yi, t, p2);
          r32_fwd<LOGN>(xab, X, t, twf, p, p2);
          // park A-hat in the residue area and B-hat in plane 1, which the
          // one-vector inverse exchanges never touch; thread-private slots
          // [e T + t], read back only by their owner
          __syncthreads();  // every read of plane 1 by the last forward exchange is done
#pragma unroll
          for (int e = 0; e < 32; e++) {
            Park[e * C::T + t] = xab[0][e];
            X[N + e * C::T + t] = xab[1][e];
          }
        }
#pragma unroll 1
        for (int P = P0; P < 3; P++) {
          // P = 0: A-hat^2, 1: B-hat^2, 2: A-hat B-hat
          const uint32_t* U = (P == 1 ? X + N : Park) + t;
          const uint32_t* V = (P == 0 ? Park : X + N) + t;
          uint32_t x[1][32];
#pragma unroll
          for (int e = 0; e < 32; e++) x[0][e] = mont(U[e * C::T], V[e * C::T], p, pinv);
          r32_inv<LOGN>(x, X, t, twi, p, p2);
          uint32_t* g = G9 + (3 * P + j) * M;
#pragma unroll
          for (int e = 0; e < 16; e++) g[t + e * (N / 32)] = x[0][e];
        }
      }
      if (phase == 0) {
        //                 G     ADD    AWS    OWS
        r32_epilogue<LOGN, true, true, false, true>(X, G9 + 0 * M, agg, t, b + inst * M, t1);  // a^2 + b
        r32_epilogue<LOGN, true, true, false, true>(X, G9 + 3 * M, agg, t, b + inst * M, t2);  // b^2 + b
        r32_epilogue<LOGN, true, false, false, true>(X, G9 + 6 * M, agg, t, nullptr, t3);       // a b
      } else {
        r32_epilogue<LOGN, true, true, true, false>(X, G9 + 6 * M, agg, t, t3, out + inst * M);  // t1 t2 + t3
      }
    }
  }
}

// ------------------------------------------------------------ beyond one CTA
// N = 2^15, 2^16 (512K / 1M-bit operands): one instance per
// thread-block cluster of CR = N / 16384 CTAs of 1024 threads x 16 register
// elements; global thread gt = rank * 1024 + tid runs exactly the register
// passes of the one-CTA kernel (the passes only see gt).  Exchanges go
// through distributed shared memory: the writer stores each element into the
// CTA (and slot e * 1024 + tid) of the thread that reads it in the next
// layout, then a cluster barrier, then purely local, conflict-free reads.
// With LOGN - 4(P+1) low bits per pass, the CTA-rank bits of gt land on the
// top index bits in every layout but pass 0's, so only the pass 0 <-> 1
// exchanges move data between CTAs.  Residues are stored with consecutive
// ownership (CTA r owns coefficients [r M/CR, (r+1) M/CR)), so the CRT,
// aggregation and L / H publish are local except one 8-word H spill per CTA,
// and the resolve is the cluster-wide carry scan.
template <int LOGN, int T_>
struct NttClCfg {
  static constexpr int N = 1 << LOGN, M = N / 2, T = T_;
  static constexpr int LT = T == 1024 ? 10 : (T == 512 ? 9 : 8);  // log2 T
  static constexpr int CR = N / (T * 16);
  static constexpr int LB = LT + 4;   // local index bits of a CTA's slice
  static constexpr int PL = T * 16;   // words of one exchange plane per CTA
  static constexpr int MS = M / CR;   // coefficients / limbs owned by a CTA
  static constexpr int SMEM_WORDS = 2 * PL + 3 * MS + 32 + 2 * CR;
  static constexpr int MINB = T <= 512 ? BN_NTT_CL_MINB : 1;
  static_assert(CR >= 2 && CR <= 8 && MS == 8 * T && (1 << LT) == T, "cluster layout");
  static_assert(PassCfg<LOGN, 1>::LO <= LT, "rank bits must sit on top of the index from pass 1 on");
};

template <int LO>
BN_DEV int unlay_t(int u) { return (u & ((1 << LO) - 1)) | ((u >> (LO + 4)) << LO); }

template <int LOGN, int T, int LO_FROM, int LO_TO, int NV, class Cluster>
BN_DEV void xchg_cl(uint32_t (&x)[NV][16], uint32_t* X0, int gt, Cluster& cl) {
  using C = NttClCfg<LOGN, T>;
  cl.sync();  // every reader of every CTA's planes is done
  const uint32_t x0 = smem_addr(X0);
#pragma unroll
  for (int e = 0; e < 16; e++) {
    const int u = lay<LO_FROM>(gt, e);
    const int gto = unlay_t<LO_TO>(u);
    const int eto = (u >> LO_TO) & 15;
    const uint32_t dst = mapa_rank(x0 + 4 * (eto * C::T + (gto & (C::T - 1))), gto / C::T);
#pragma unroll
    for (int v = 0; v < NV; v++) st_cluster(dst + 4 * v * C::PL, x[v][e]);
  }
  cl.sync();
#pragma unroll
  for (int v = 0; v < NV; v++)
#pragma unroll
    for (int e = 0; e < 16; e++) x[v][e] = X0[v * C::PL + e * C::T + threadIdx.x];
}

// Passes 1..3 keep the CTA-rank bits of gt on the top index bits, so their
// exchanges are CTA-local and are exactly the one-CTA 2^14-point exchanges
// (same LO values, local thread id, swizzled plane, __syncthreads); only
// pass 0 <-> 1 goes through DSMEM.
template <int LOGN, int T, int NV, class Cluster>
BN_DEV void fwd_all_cl(uint32_t (&x)[NV][16], uint32_t* X0, int gt, const uint2* tw, uint32_t p, uint32_t p2,
                       Cluster& cl) {
  using C = NttClCfg<LOGN, T>;
  constexpr int L0 = PassCfg<LOGN, 0>::LO, L1 = PassCfg<LOGN, 1>::LO, L2 = PassCfg<LOGN, 2>::LO,
                L3 = PassCfg<LOGN, 3>::LO;
  const int tid = threadIdx.x;
  fwd_pass<LOGN, 0, true, NV>(x, gt, tw, p, p2);
  xchg_cl<LOGN, T, L0, L1, NV>(x, X0, gt, cl);
  fwd_pass<LOGN, 1, true, NV>(x, gt, tw, p, p2);
  xchg<C::LB, L1, L2, T, NV, C::PL>(x, X0, 0, tid);
  fwd_pass<LOGN, 2, true, NV>(x, gt, tw, p, p2);
  if constexpr (LOGN > 12) {
    xchg<C::LB, L2, L3, T, NV, C::PL>(x, X0, 0, tid);
    fwd_pass<LOGN, 3, true, NV>(x, gt, tw, p, p2);
  }
}

template <int LOGN, int T, class Cluster>
BN_DEV void inv_all_cl(uint32_t (&x1)[16], uint32_t* X0, int gt, const uint2* tw, uint32_t p, uint32_t p2,
                       Cluster& cl) {
  using C = NttClCfg<LOGN, T>;
  constexpr int L0 = PassCfg<LOGN, 0>::LO, L1 = PassCfg<LOGN, 1>::LO, L2 = PassCfg<LOGN, 2>::LO,
                L3 = PassCfg<LOGN, 3>::LO;
  const int tid = threadIdx.x;
  uint32_t(&x)[1][16] = reinterpret_cast<uint32_t(&)[1][16]>(x1);
  if constexpr (LOGN > 12) {
    inv_pass<LOGN, 3>(x1, gt, tw, p, p2);
    xchg<C::LB, L3, L2, T, 1, C::PL>(x, X0, 0, tid);
  }
  inv_pass<LOGN, 2>(x1, gt, tw, p, p2);
  xchg<C::LB, L2, L1, T, 1, C::PL>(x, X0, 0, tid);
  inv_pass<LOGN, 1>(x1, gt, tw, p, p2);
  xchg_cl<LOGN, T, L1, L0, 1>(x, X0, gt, cl);
  inv_pass<LOGN, 0>(x1, gt, tw, p, p2);
}

template <int LOGN, int T>
__global__ void __launch_bounds__(T, NttClCfg<LOGN, T>::MINB)
    mul_ntt_cluster_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                           const uint2* __restrict__ tw) {
  using C = NttClCfg<LOGN, T>;
  constexpr int N = C::N, M = C::M, MS = C::MS;
  extern __shared__ __align__(16) uint32_t sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const int gt = rank * C::T + tid;
  uint32_t* X0 = sm;                  // plane 0 | plane 1
  uint32_t* Res = sm + 2 * C::PL;     // 3 x MS, consecutive ownership
  uint32_t* agg = Res + 3 * MS;       // 32
  uint32_t* cta_agg = agg + 32;       // 2 CR
  const uint64_t n_cl = gridDim.x / C::CR;
  int parity = 0;
  for (uint64_t inst = blockIdx.x / C::CR; inst < n_inst; inst += n_cl, parity ^= 1) {
    const uint32_t* ai = a + inst * M;
    const uint32_t* bi = b + inst * M;
#pragma unroll 1
    for (int j = 0; j < kNumPrimes; j++) {
      const uint32_t p = c_pc[j].p, p2 = c_pc[j].p2, pinv = c_pc[j].pinv;
      const uint2* twf = tw + (2 * j + 0) * (N - 1);
      const uint2* twi = tw + (2 * j + 1) * (N - 1);
      uint32_t xab[2][16];
#pragma unroll
      for (int e = 0; e < 8; e++) {
        xab[0][e] = red2(red2(__ldg(ai + gt + e * (N / 16)), p2), p2);
        xab[1][e] = red2(red2(__ldg(bi + gt + e * (N / 16)), p2), p2);
      }
#pragma unroll
      for (int e = 8; e < 16; e++) xab[0][e] = xab[1][e] = 0u;
      fwd_all_cl<LOGN, T, 2>(xab, X0, gt, twf, p, p2, cl);
      uint32_t x[16];
#pragma unroll
      for (int e = 0; e < 16; e++) x[e] = mont(xab[0][e], xab[1][e], p, pinv);
      inv_all_cl<LOGN, T>(x, X0, gt, twi, p, p2, cl);
      // coefficient k = gt + e N/16 (e < 8) -> its owner's residue array
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const int k = gt + e * (N / 16);
        st_cluster(mapa_rank(smem_addr(Res + j * MS + cswz<8, false>(k & (MS - 1))), k / MS), x[e]);
      }
    }
    cl.sync();  // residues in place; every plane read is done

    // N-5 / N-6 on this CTA's consecutive coefficients [rank MS + 8 tid, +8)
    {
      uint32_t lows[8], hs[8], h0, h1;
      crt_aggregate<8, false>(Res, MS, 8 * tid, c_crt[LOGN], lows, h0, h1);
#pragma unroll
      for (int q = 0; q < 8; q++) hs[q] = q == 0 ? h0 : (q == 1 ? h1 : 0u);
      // L = plane 0 [0, MS), H = plane 1 [0, MS) (planes are dead), cswz<8>
      uint32_t* L = X0;
      uint32_t* H = X0 + C::PL;
      sts_swz<8, 8, false>(L, 8 * tid, lows);
      if (tid < C::T - 1) {
        sts_swz<8, 8, false>(H, 8 * tid + 8, hs);
      } else {
        // the CTA's top chunk spills into the next CTA's H[0, 8); the
        // instance's top chunk wraps to zero CTA 0's H[0, 8)
        if (rank == C::CR - 1) {
#pragma unroll
          for (int q = 0; q < 8; q++) hs[q] = 0;
        }
        const uint32_t dst = mapa_rank(smem_addr(H), (rank + 1) % C::CR);
#pragma unroll
        for (int q = 0; q < 8; q++) st_cluster(dst + 4 * cswz<8, false>(q), hs[q]);
      }
    }
    cl.sync();
    // N-7: R = L + H across the cluster, store
    {
      uint32_t xl[8], yh[8], r[8], g, pp;
      lds_swz<8, 8, false>(xl, X0, 8 * tid);
      lds_swz<8, 8, false>(yh, X0 + C::PL, 8 * tid);
      chunk_sum<8>(xl, yh, r, g, pp);
      const uint32_t cin = cluster_carry_scan<C::CR>(g, pp, agg, cta_agg, parity, cl);
      chunk_apply<8>(xl, r, cin);
      store_limbs<8>(out + inst * M + (uint64_t)rank * MS + 8 * tid, r);
    }
  }
}

template <int LOGN, int T>
static cudaError_t launch_ntt_cluster_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                        const NttTables& tb, cudaStream_t st, int n_sm) {
  using C = NttClCfg<LOGN, T>;
  constexpr size_t smem = C::SMEM_WORDS * sizeof(uint32_t);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(C::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::CR;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(C::CR);
  static LaunchCache cache;
  int max_cl = 0;
  cudaError_t e = cached_query(cache, [&](int* o) {
    cudaError_t e1 = cudaFuncSetAttribute(mul_ntt_cluster_kernel<LOGN, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e1 != cudaSuccess) return e1;
    return cudaOccupancyMaxActiveClusters(o, mul_ntt_cluster_kernel<LOGN, T>, &cfg);
  }, &max_cl);
  if (e != cudaSuccess) return e;
  if (max_cl < 1) return cudaErrorInvalidConfiguration;
  uint64_t n_cl = n_inst < (uint64_t)max_cl ? n_inst : (uint64_t)max_cl;
  n_cl = cap_grid((unsigned)n_cl);
  cfg.gridDim = dim3((unsigned)(n_cl * C::CR));
  e = cudaLaunchKernelEx(&cfg, mul_ntt_cluster_kernel<LOGN, T>, out, a, b, n_inst, tb.tw);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Cluster version of the 32-element kernel (2^19, 2^20 bits): T = 512
// threads x 32 elements per CTA, CR = N / 16384 CTAs (2 / 4).  Same
// structure as mul_ntt_cluster_kernel — only pass 0 <-> 1 crosses CTAs
// (DSMEM), later exchanges are the local conflict-free xchg32 over the CTA's
// 2^14-word slice — with 128 registers and one fewer exchange per transform.
template <int LOGN>
struct NttCl32Cfg {
  static constexpr int N = 1 << LOGN, M = N / 2, T = 512, LT = 9;
  static constexpr int CR = N / (T * 32);
  static constexpr int PL = T * 32;  // 16384
  static constexpr int MS = M / CR;  // 8192 = 16 T
  static constexpr int NP = (LOGN + 4) / 5;
  static constexpr int SMEM_WORDS = 2 * PL + 3 * MS + T / 32 + 2 * CR;
  static_assert(CR >= 2 && CR <= 8 && MS == 16 * T, "cluster32 layout");
  static_assert(PassCfgR<LOGN, 1, 5>::LO <= LT, "rank bits on top from pass 1 on");
};

// The last forward DIF stage and the first inverse DIT stage (stage
// log2 N - 1: index pairs (i, i ^ 1)) have twiddle 1, so together with the
// pointwise product between them they are a 2-point cyclic convolution of
// each pair: with A' = (a0 + a1, a0 - a1), B' likewise, C' = A' B'
// (Montgomery) and c = (C'0 + C'1, C'0 - C'1):  c0 = S + D, c1 = S - D,
// S = (a0 + a1)(b0 + b1), D = (a0 - a1)(b0 - b1) — the same lazy-reduced
// operations in the same order as fwd_pass / mont / inv_pass on that stage.
// In a layout whose lowest register-free index bit is bit 0 (LO = 1) the
// partner of every element sits in lane ^ 1, so one shuffle per value
// replaces the exchange into and out of the bit-0 layout.  Lane bit 0 = 0
// keeps c0, lane bit 0 = 1 keeps c1.
BN_DEV void pair_conv_shfl(const uint32_t (&xab)[2][32], uint32_t (&x)[32], uint32_t p, uint32_t p2,
                           uint32_t pinv) {
  const bool hi = threadIdx.x & 1;
#pragma unroll
  for (int e = 0; e < 32; e++) {
    const uint32_t ao = __shfl_xor_sync(0xFFFFFFFFu, xab[0][e], 1);
    const uint32_t bo = __shfl_xor_sync(0xFFFFFFFFu, xab[1][e], 1);
    const uint32_t a0 = hi ? ao : xab[0][e], a1 = hi ? xab[0][e] : ao;
    const uint32_t b0 = hi ? bo : xab[1][e], b1 = hi ? xab[1][e] : bo;
    const uint32_t S = mont(red2(a0 + a1, p2), red2(b0 + b1, p2), p, pinv);
    const uint32_t D = mont(red2(a0 - a1 + p2, p2), red2(b0 - b1 + p2, p2), p, pinv);
    x[e] = hi ? S - D + p2 : S + D;
  }
}

template <int LO>
BN_DEV int unlay32_t(int u) { return (u & ((1 << LO) - 1)) | ((u >> (LO + 5)) << LO); }

template <int LOGN, int LO_FROM, int LO_TO, int NV, class Cluster>
BN_DEV void xchg_cl32(uint32_t (&x)[NV][32], uint32_t* X0, int gt, Cluster& cl) {
  using C = NttCl32Cfg<LOGN>;
  cl.sync();
  const uint32_t x0 = smem_addr(X0);
#pragma unroll
  for (int e = 0; e < 32; e++) {
    const int u = lay32<LO_FROM>(gt, e);
    const int gto = unlay32_t<LO_TO>(u);
    const int eto = (u >> LO_TO) & 31;
    const uint32_t dst = mapa_rank(x0 + 4 * (eto * C::T + (gto & (C::T - 1))), gto >> C::LT);
#pragma unroll
    for (int v = 0; v < NV; v++) st_cluster(dst + 4 * v * C::PL, x[v][e]);
  }
  cl.sync();
#pragma unroll
  for (int v = 0; v < NV; v++)
#pragma unroll
    for (int e = 0; e < 32; e++) x[v][e] = X0[v * C::PL + e * C::T + threadIdx.x];
}

template <int LOGN>
__global__ void __launch_bounds__(512, 1)
    mul_ntt_cluster32_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                             const uint2* __restrict__ tw) {
  using C = NttCl32Cfg<LOGN>;
  constexpr int N = C::N, M = C::M, MS = C::MS, PL = C::PL;
  constexpr int L0 = PassCfgR<LOGN, 0, 5>::LO, L1 = PassCfgR<LOGN, 1, 5>::LO, L2 = PassCfgR<LOGN, 2, 5>::LO;
  constexpr int L3 = PassCfgR<LOGN, 3, 5>::LO;
  extern __shared__ __align__(16) uint32_t sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const int gt = rank * C::T + tid;
  uint32_t* X0 = sm;
  uint32_t* Res = sm + 2 * PL;
  uint32_t* agg = Res + 3 * MS;
  uint32_t* cta_agg = agg + C::T / 32;
  const uint64_t n_cl = gridDim.x / C::CR;
  int parity = 0;
  for (uint64_t inst = blockIdx.x / C::CR; inst < n_inst; inst += n_cl, parity ^= 1) {
    const uint32_t* ai = a + inst * M;
    const uint32_t* bi = b + inst * M;
#pragma unroll 1
    for (int j = 0; j < kNumPrimes; j++) {
      const uint32_t p = c_pc[j].p, p2 = c_pc[j].p2, pinv = c_pc[j].pinv;
      const uint2* twf = tw + (2 * j + 0) * (N - 1);
      const uint2* twi = tw + (2 * j + 1) * (N - 1);
      uint32_t xab[2][32];
#pragma unroll
      for (int e = 0; e < 16; e++) {
        xab[0][e] = red2(red2(__ldg(ai + gt + e * (N / 32)), p2), p2);
        xab[1][e] = red2(red2(__ldg(bi + gt + e * (N / 32)), p2), p2);
      }
#pragma unroll
      for (int e = 16; e < 32; e++) xab[0][e] = xab[1][e] = 0u;
      fwd_pass<LOGN, 0, true, 2, 32>(xab, gt, twf, p, p2);
      xchg_cl32<LOGN, L0, L1, 2>(xab, X0, gt, cl);
      fwd_pass<LOGN, 1, true, 2, 32>(xab, gt, twf, p, p2);
      xchg32<L1, L2, 2, PL>(xab, X0, tid);
      fwd_pass<LOGN, 2, true, 2, 32>(xab, gt, twf, p, p2);
      uint32_t x[1][32];
      if constexpr (C::NP > 3 && BN_NTT_PAIR_CONV) {
        // 2^16: the one-stage pass 3 (bit 0) collapses into a 2-point
        // convolution across lane pairs (pair_conv_shfl): no pass-3 layout,
        // two exchanges fewer per prime
        pair_conv_shfl(xab, x[0], p, p2, pinv);
      } else {
        if constexpr (C::NP > 3) {
          xchg32<L2, L3, 2, PL>(xab, X0, tid);
          fwd_pass<LOGN, 3, true, 2, 32>(xab, gt, twf, p, p2);
        }
#pragma unroll
        for (int e = 0; e < 32; e++) x[0][e] = mont(xab[0][e], xab[1][e], p, pinv);
        if constexpr (C::NP > 3) {
          inv_pass<LOGN, 3, 32>(x[0], gt, twi, p, p2);
          xchg32<L3, L2, 1, PL>(x, X0, tid);
        }
      }
      inv_pass<LOGN, 2, 32>(x[0], gt, twi, p, p2);
      xchg32<L2, L1, 1, PL>(x, X0, tid);
      inv_pass<LOGN, 1, 32>(x[0], gt, twi, p, p2);
      xchg_cl32<LOGN, L1, L0, 1>(x, X0, gt, cl);
      inv_pass<LOGN, 0, 32>(x[0], gt, twi, p, p2);
      // coefficient k = gt + e N/32 (e < 16) -> its owner's residue array
#pragma unroll
      for (int e = 0; e < 16; e++) {
        const int k = gt + e * (N / 32);
        st_cluster(mapa_rank(smem_addr(Res + j * MS + cswz<16>(k & (MS - 1))), k / MS), x[0][e]);
      }
    }
    cl.sync();
    // CRT / aggregate 16 consecutive coefficients [rank MS + 16 tid, +16)
    {
      uint32_t lows[16], hs[16], h0, h1;
      crt_aggregate<16, true>(Res, MS, 16 * tid, c_crt[LOGN], lows, h0, h1);
#pragma unroll
      for (int q = 0; q < 16; q++) hs[q] = q == 0 ? h0 : (q == 1 ? h1 : 0u);
      uint32_t* L = X0;
      uint32_t* H = X0 + PL;
      sts_swz<16, 16>(L, 16 * tid, lows);
      if (tid < C::T - 1) {
        sts_swz<16, 16>(H, 16 * tid + 16, hs);
      } else {
        if (rank == C::CR - 1) {
#pragma unroll
          for (int q = 0; q < 16; q++) hs[q] = 0;
        }
        const uint32_t dst = mapa_rank(smem_addr(H), (rank + 1) % C::CR);
#pragma unroll
        for (int q = 0; q < 16; q++) st_cluster(dst + 4 * cswz<16>(q), hs[q]);
      }
    }
    cl.sync();
    {
      uint32_t xl[16], yh[16], r[16], g, pp;
      lds_swz<16, 16>(xl, X0, 16 * tid);
      lds_swz<16, 16>(yh, X0 + PL, 16 * tid);
      chunk_sum<16>(xl, yh, r, g, pp);
      const uint32_t cin = cluster_carry_scan<C::CR>(g, pp, agg, cta_agg, parity, cl);
      chunk_apply<16>(xl, r, cin);
      store_limbs<16>(out + inst * M + (uint64_t)rank * MS + 16 * tid, r);
    }
  }
}

template <int LOGN>
static cudaError_t launch_ntt_cluster32_t(uint32_t* out, const uint32_t* a, const uint32_t* b,
                                          uint64_t n_inst, const NttTables& tb, cudaStream_t st) {
  using C = NttCl32Cfg<LOGN>;
  constexpr size_t smem = C::SMEM_WORDS * sizeof(uint32_t);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(C::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::CR;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(C::CR);
  static LaunchCache cache;
  int max_cl = 0;
  cudaError_t e = cached_query(cache, [&](int* o) {
    cudaError_t e1 = cudaFuncSetAttribute(mul_ntt_cluster32_kernel<LOGN>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e1 != cudaSuccess) return e1;
    return cudaOccupancyMaxActiveClusters(o, mul_ntt_cluster32_kernel<LOGN>, &cfg);
  }, &max_cl);
  if (e != cudaSuccess) return e;
  if (max_cl < 1) return cudaErrorInvalidConfiguration;
  uint64_t n_cl = n_inst < (uint64_t)max_cl ? n_inst : (uint64_t)max_cl;
  n_cl = cap_grid((unsigned)n_cl);
  cfg.gridDim = dim3((unsigned)(n_cl * C::CR));
  e = cudaLaunchKernelEx(&cfg, mul_ntt_cluster32_kernel<LOGN>, out, a, b, n_inst, tb.tw);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ------------------------------------------------------------ full product
// Wide (untruncated) product: out[k] = a[k] * b[k] as 2m
// limbs.  The N = 2m point transform already yields every coefficient
// c_0..c_{2m-2} of Eq. 1 without truncation (P:338-342 with k < 2M), so the
// wide product is the same three transforms per prime keeping all 16
// register elements (e < 16) through the CRT; each thread then aggregates
// 16 consecutive coefficients into 16 lows + 2 overflow words, publishes
// them as L / H over 2m words (reading R8 with M -> 2M) and the scan-add
// resolves 2m limbs.  Shared memory: the two exchange planes + 3N residues
// per slot, so N <= 2^13 (inputs up to 128K bits, results up to 256K).
template <int LOGN>
struct NttWideCfg {
  using B = NttCfg<LOGN>;
  static constexpr int RS = 3 * B::N + (B::TPI < 32 ? 16 : 0);
  static constexpr int SMEM_WORDS = 2 * B::XW + B::IPB * RS + B::T / 32;
  // residency: up to 2^8 points a target of BN_NTT_WIDE_THREADS threads per
  // SM, bounded by what shared memory admits (A/B, ms per paper batch, 768
  // vs <= 128 registers: 1K 2.800 -> 2.755, 2K 2.966 -> 2.909, 4K 3.233 ->
  // 3.186; from 2^9 points 80 registers spill and lose: 8K 4.04 -> 4.43)
  static constexpr int BY_SMEM = (227 * 1024) / (SMEM_WORDS * 4);
  static constexpr int BY_THR = BN_NTT_WIDE_THREADS / B::T;
  static constexpr int MINB = LOGN > 8 ? (LOGN <= 12 ? 2 : 1)  // <= 128 registers
                                       : (BY_THR < 1 ? 1 : (BY_THR < BY_SMEM ? BY_THR : (BY_SMEM < 1 ? 1 : BY_SMEM)));
};

template <int LOGN>
__global__ void __launch_bounds__(NttCfg<LOGN>::T, NttWideCfg<LOGN>::MINB)
    mul_wide_ntt_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                        const uint2* __restrict__ tw) {
  using C = NttCfg<LOGN>;
  using W = NttWideCfg<LOGN>;
  constexpr int N = C::N, M = C::M, TPI = C::TPI;
  extern __shared__ __align__(16) uint32_t sm[];
  const int slot = threadIdx.x / TPI;
  const int t = threadIdx.x % TPI;
  uint32_t* X = sm + slot * (C::XW / C::IPB);  // plane-0 region of the slot
  uint32_t* X1 = X + C::XW;                      // plane-1 region of the slot
  uint32_t* Res = sm + 2 * C::XW + slot * W::RS;
  uint32_t* agg = sm + 2 * C::XW + C::IPB * W::RS;

  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  for (uint64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const uint64_t inst = grp * C::IPB + slot;
    const bool valid = inst < n_inst;
    const uint32_t* ai = a + (valid ? inst : 0) * M;
    const uint32_t* bi = b + (valid ? inst : 0) * M;

#pragma unroll 1
    for (int j = 0; j < kNumPrimes; j++) {
      const uint32_t p = c_pc[j].p, p2 = c_pc[j].p2, pinv = c_pc[j].pinv;
      const uint2* twf = tw + (2 * j + 0) * (N - 1);
      const uint2* twi = tw + (2 * j + 1) * (N - 1);
      uint32_t xab[2][16];
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const uint32_t va = valid ? __ldg(ai + t + e * (N / 16)) : 0u;
        const uint32_t vb = valid ? __ldg(bi + t + e * (N / 16)) : 0u;
        xab[0][e] = red2(red2(va, p2), p2);
        xab[1][e] = red2(red2(vb, p2), p2);
      }
#pragma unroll
      for (int e = 8; e < 16; e++) xab[0][e] = xab[1][e] = 0u;
      fwd_all<LOGN, true, 2>(xab, sm, slot * N, t, twf, p, p2);
      uint32_t x[16];
#pragma unroll
      for (int e = 0; e < 16; e++) x[e] = mont(xab[0][e], xab[1][e], p, pinv);
      inv_all<LOGN>(x, sm, slot * N, t, twi, p, p2);
      // all N coefficients (the last, c_{N-1}, is 0)
#pragma unroll
      for (int e = 0; e < 16; e++) Res[j * N + cswz<16>(t + e * (N / 16))] = x[e];
    }
    bar<TPI>();

    // Garner CRT of 16 consecutive coefficients, aggregate, publish; the
    // planes are dead (the last exchange read them before the barrier above):
    // L = plane 0 region, H = plane 1 region, N words each
    {
      uint32_t lows[16], h0, h1;
      crt_aggregate<16, true>(Res, N, 16 * t, c_crt[LOGN], lows, h0, h1);
      publish_lh<16, true>(X, X1, 16 * t, N, lows, h0, h1);
    }
    bar<TPI>();
    {
      uint32_t xl[16], yh[16], r[16];
      lds_swz<16, 16>(xl, X, 16 * t);
      lds_swz<16, 16>(yh, X1, 16 * t);
      add_regs<16, TPI>(xl, yh, r, valid, agg);
      if (valid) store_limbs<16>(out + inst * N + 16 * t, r);
    }
    __syncthreads();
  }
}

// Wide product at 2^18 bits (N = 2^14 points, 2^15-limb result) in ONE CTA
// of 512 threads x 32 register elements: the 16-element wide kernel keeps
// 3 N raw residues (192 KiB) beside two exchange planes, which does not fit.
// Here the forward transforms of a and b go one after the other through a
// single plane (A-hat held in registers meanwhile) and Garner runs
// incrementally, element by element in the pass-0 layout, so each thread only
// ever touches its own coefficients until the aggregation:
//   prime 0: R0[k] = r0;  prime 1: T1[k] = t1(y1, r0);
//   prime 2: c = r0 + p0 t1 + p0 p1 t2 -> C0[k] | C1[k] | C2[k] (3 words)
// in the three N-word regions (plane, R0, T1), then thread t aggregates the
// 32 consecutive coefficients [32 t, 32 t + 32), publishes L / H (reading R8
// with M -> 2M) and resolves all N = 2m limbs: 3 N words = 192 KiB.
// The c regions use the 32-word-per-thread swizzle (chunk ^ row & 7): the
// pass-layout writes and the 32-consecutive reads are both conflict free.
BN_DEV int cswz32(int k) { return k ^ (((k >> 5) & 7) << 2); }

template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 32, 1)
    mul_wide_ntt_r32_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                            const uint2* __restrict__ tw) {
  constexpr int N = 1 << LOGN, M = N / 2, T = N / 32;
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* P0 = sm;          // exchange plane, later C0 / L
  uint32_t* R0 = sm + N;      // r0, later C1 / H
  uint32_t* T1 = sm + 2 * N;  // t1, later C2
  uint32_t* agg = sm + 3 * N;
  const int t = threadIdx.x;
  const CrtConst& k = c_crt[LOGN];
  const uint32_t q0 = c_pc[0].p, q1 = c_pc[1].p, q2 = c_pc[2].p;
  for (uint64_t inst = blockIdx.x; inst < n_inst; inst += gridDim.x) {
    const uint32_t* ai = a + inst * M;
    const uint32_t* bi = b + inst * M;
#pragma unroll 1
    for (int j = 0; j < kNumPrimes; j++) {
      const uint32_t p = c_pc[j].p, p2 = c_pc[j].p2, pinv = c_pc[j].pinv;
      const uint2* twf = tw + (2 * j + 0) * (N - 1);
      const uint2* twi = tw + (2 * j + 1) * (N - 1);
      // a, then b, through ONE inlined copy of the forward transform (two
      // copies spilled more: ptxas -v); A-hat is kept while b is transformed
      uint32_t xa[1][32], xb[1][32];
#pragma unroll 1
      for (int v = 0; v < 2; v++) {
        const uint32_t* src = v ? bi : ai;
#pragma unroll
        for (int e = 0; e < 16; e++) xb[0][e] = red2(red2(__ldg(src + t + e * (N / 32)), p2), p2);
#pragma unroll
        for (int e = 16; e < 32; e++) xb[0][e] = 0u;
        r32_fwd1<LOGN>(xb, P0, t, twf, p, p2);
        if (v == 0) {
#pragma unroll
          for (int e = 0; e < 32; e++) xa[0][e] = xb[0][e];
        }
      }
#pragma unroll
      for (int e = 0; e < 32; e++) xa[0][e] = mont(xa[0][e], xb[0][e], p, pinv);
      r32_inv<LOGN>(xa, P0, t, twi, p, p2);
      // incremental Garner on this thread's own coefficients k = t + e N/32
      if (j == 0) {
#pragma unroll
        for (int e = 0; e < 32; e++) R0[t + e * (N / 32)] = red2(shoup(xa[0][e], k.k0, k.k0_sh, q0), q0);
      } else if (j == 1) {
#pragma unroll
        for (int e = 0; e < 32; e++) {
          const uint32_t r0 = R0[t + e * (N / 32)];
          const uint32_t u = shoup(xa[0][e], k.k1i, k.k1i_sh, q1);
          const uint32_t v = shoup(r0, k.i01, k.i01_sh, q1);
          T1[t + e * (N / 32)] = red2(red2(u + 2 * q1 - v, 2 * q1), q1);
        }
      } else {
        __syncthreads();  // every read of the plane by the last inverse exchange is done
#pragma unroll
        for (int e = 0; e < 32; e++) {
          const int kk = t + e * (N / 32);
          const uint32_t r0 = R0[kk], t1 = T1[kk];
          const uint32_t a2v = shoup(xa[0][e], k.k2i, k.k2i_sh, q2);
          const uint32_t b2v = shoup(r0, k.i012, k.i012_sh, q2);
          const uint32_t c2v = shoup(t1, k.p0i012, k.p0i012_sh, q2);
          const uint32_t d = red2(b2v + c2v, 2 * q2);
          const uint32_t t2 = red2(red2(a2v + 2 * q2 - d, 2 * q2), q2);
          const uint64_t v64 = (uint64_t)q0 * t1 + r0;
          const uint64_t w = (uint64_t)k.p01_lo * t2 + v64;
          const uint64_t hh = (uint64_t)k.p01_hi * t2 + (w >> 32);
          const int ks = cswz32(kk);
          P0[ks] = (uint32_t)w;
          R0[ks] = (uint32_t)hh;
          T1[ks] = (uint32_t)(hh >> 32);
        }
      }
    }
    __syncthreads();
    // aggregate the 32 consecutive coefficients [32 t, 32 t + 32)
    uint32_t lows[32], h0, h1;
    {
      uint32_t a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
      for (int c = 0; c < 8; c++) {
        const int ks = cswz32(32 * t + 4 * c);
        const uint4 w0 = *reinterpret_cast<const uint4*>(P0 + ks);
        const uint4 w1 = *reinterpret_cast<const uint4*>(R0 + ks);
        const uint4 w2 = *reinterpret_cast<const uint4*>(T1 + ks);
        const uint32_t c0[4] = {w0.x, w0.y, w0.z, w0.w}, c1[4] = {w1.x, w1.y, w1.z, w1.w},
                       c2[4] = {w2.x, w2.y, w2.z, w2.w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
          add3(a0, a1, a2, c0[q], c1[q], c2[q]);
          lows[4 * c + q] = a0;
          a0 = a1;
          a1 = a2;
          a2 = 0;
        }
      }
      h0 = a0;
      h1 = a1;
    }
    __syncthreads();  // every read of C0..C2 is done
    // publish: L = P0 region, H = R0 region (N words each, cswz32 layout)
    {
#pragma unroll
      for (int c = 0; c < 8; c++)
        *reinterpret_cast<uint4*>(P0 + cswz32(32 * t + 4 * c)) =
            make_uint4(lows[4 * c], lows[4 * c + 1], lows[4 * c + 2], lows[4 * c + 3]);
      const int hb = t + 1 < T ? 32 * t + 32 : 0;  // the top chunk zeroes H[0, 32) (positions >= N dropped)
      const uint32_t g0 = t + 1 < T ? h0 : 0u, g1 = t + 1 < T ? h1 : 0u;
#pragma unroll
      for (int c = 0; c < 8; c++)
        *reinterpret_cast<uint4*>(R0 + cswz32(hb + 4 * c)) =
            make_uint4(c == 0 ? g0 : 0u, c == 0 ? g1 : 0u, 0u, 0u);
    }
    __syncthreads();
    // resolve R = L + H over the N = 2m limbs, 32 per thread
    {
      uint32_t x[32], y[32];
#pragma unroll
      for (int c = 0; c < 8; c++) {
        const int ks = cswz32(32 * t + 4 * c);
        const uint4 l = *reinterpret_cast<const uint4*>(P0 + ks);
        const uint4 h = *reinterpret_cast<const uint4*>(R0 + ks);
        x[4 * c] = l.x; x[4 * c + 1] = l.y; x[4 * c + 2] = l.z; x[4 * c + 3] = l.w;
        y[4 * c] = h.x; y[4 * c + 1] = h.y; y[4 * c + 2] = h.z; y[4 * c + 3] = h.w;
      }
      add_regs_inplace<32, T>(x, y, true, agg);
      store_limbs<32>(out + inst * N + 32 * t, x);
    }
    __syncthreads();  // regions / agg reused by the next instance
  }
}

template <int LOGN>
static cudaError_t launch_wide_ntt_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                     const NttTables& tb, cudaStream_t st, int n_sm) {
  if constexpr (LOGN == 14) {
    constexpr int T = (1 << LOGN) / 32;
    constexpr size_t smem = (3 * (1 << LOGN) + T / 32) * sizeof(uint32_t);
    static LaunchCache cache;
    int per_sm = 0;
    cudaError_t e = resident_ctas(cache, mul_wide_ntt_r32_kernel<LOGN>, T, smem, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint64_t cap = (uint64_t)n_sm * per_sm;
    const unsigned grid = cap_grid((unsigned)(n_inst < cap ? n_inst : cap));
    mul_wide_ntt_r32_kernel<LOGN><<<grid, T, smem, st>>>(out, a, b, n_inst, tb.tw);
    return cudaGetLastError();
  } else if constexpr (LOGN > 13) {
    return cudaErrorInvalidValue;
  } else {
    using C = NttCfg<LOGN>;
    constexpr size_t smem = NttWideCfg<LOGN>::SMEM_WORDS * sizeof(uint32_t);
    static LaunchCache cache;
    int per_sm = 0;
    cudaError_t e = resident_ctas(cache, mul_wide_ntt_kernel<LOGN>, C::T, smem, &per_sm);
    if (e != cudaSuccess) return e;
    const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint64_t cap = (uint64_t)n_sm * per_sm * 8;
    const unsigned grid = cap_grid((unsigned)(n_groups < cap ? n_groups : cap));
    mul_wide_ntt_kernel<LOGN><<<grid, C::T, smem, st>>>(out, a, b, n_inst, tb.tw);
    return cudaGetLastError();
  }
}

// Forward transform only (tests): rows of N residues < p, in place,
// bit-reversed output in [0, p).
template <int LOGN>
__global__ void __launch_bounds__(NttCfg<LOGN>::T)
    ntt_forward_debug_kernel(uint32_t* xg, uint64_t n_inst, const uint2* __restrict__ tw, int j) {
  using C = NttCfg<LOGN>;
  constexpr int N = C::N;
  extern __shared__ __align__(16) uint32_t sm[];
  const int slot = threadIdx.x / C::TPI;
  const int t = threadIdx.x % C::TPI;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  for (uint64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const uint64_t inst = grp * C::IPB + slot;
    const bool valid = inst < n_inst;
    uint32_t* row = xg + (valid ? inst : 0) * N;
    const uint32_t p = c_pc[j].p, p2 = c_pc[j].p2;
    uint32_t x[1][16];
#pragma unroll
    for (int e = 0; e < 16; e++) x[0][e] = valid ? row[t + e * (N / 16)] : 0u;
    fwd_all<LOGN, false, 1>(x, sm, slot * N, t, tw + 2 * j * (N - 1), p, p2);
    constexpr int LO_LAST = PassCfg<LOGN, C::NP - 1>::LO;
    if (valid) {
#pragma unroll
      for (int e = 0; e < 16; e++) row[lay<LO_LAST>(t, e)] = red2(x[0][e], p);
    }
    __syncthreads();
  }
}

template <int LOGN>
static cudaError_t launch_ntt_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                const NttTables& tb, cudaStream_t st, int n_sm) {
  using C = NttCfg<LOGN>;
  constexpr size_t smem = C::SMEM_WORDS * sizeof(uint32_t);
  static LaunchCache cache;
  int per_sm = 0;
  cudaError_t e = resident_ctas(cache, mul_ntt_kernel<LOGN>, C::T, smem, &per_sm);
  if (e != cudaSuccess) return e;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t cap = (uint64_t)n_sm * per_sm * 8;
  const unsigned grid = cap_grid((unsigned)(n_groups < cap ? n_groups : cap));
  mul_ntt_kernel<LOGN><<<grid, C::T, smem, st>>>(out, a, b, n_inst, tb.tw);
  return cudaGetLastError();
}

template <int LOGN>
static cudaError_t poly_ntt_geom_t(uint64_t n_inst, int n_sm, unsigned* grid, uint64_t* ws_words) {
  static LaunchCache cache;
  int per_sm = 0;
  if constexpr (LOGN >= BN_POLY_R32_MIN) {
    using C = NttR32Cfg<LOGN>;
    constexpr size_t smem = C::SMEM_WORDS * sizeof(uint32_t);
    cudaError_t e = resident_ctas(cache, poly_ntt_r32_kernel<LOGN>, C::T, smem, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint64_t cap = (uint64_t)n_sm * per_sm;  // one resident wave: one workspace slice each
    *grid = cap_grid((unsigned)(n_inst < cap ? n_inst : cap));
    *ws_words = (uint64_t)*grid * PolyR32Cfg<LOGN>::WS_WORDS;
  } else {
    using C = NttCfg<LOGN, kPolyNttTT>;
    constexpr size_t smem = PolyNttCfg<LOGN>::SMEM_WORDS * sizeof(uint32_t);
    cudaError_t e = resident_ctas(cache, poly_ntt_kernel<LOGN>, C::T, smem, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
    const uint64_t cap = (uint64_t)n_sm * per_sm;  // one resident wave: one workspace slice each
    *grid = cap_grid((unsigned)(n_groups < cap ? n_groups : cap));
    *ws_words = (uint64_t)*grid * C::IPB * 3 * C::M;
  }
  return cudaSuccess;
}

template <int LOGN>
static cudaError_t launch_poly_ntt_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                     const NttTables& tb, uint32_t* ws, uint64_t ws_words, cudaStream_t st,
                                     int n_sm) {
  unsigned grid = 0;
  uint64_t need = 0;
  cudaError_t e = poly_ntt_geom_t<LOGN>(n_inst, n_sm, &grid, &need);
  if (e != cudaSuccess) return e;
  if (ws_words < need) return cudaErrorInvalidValue;
  if constexpr (LOGN >= BN_POLY_R32_MIN) {
    using C = NttR32Cfg<LOGN>;
    constexpr size_t smem = C::SMEM_WORDS * sizeof(uint32_t);
    poly_ntt_r32_kernel<LOGN><<<grid, C::T, smem, st>>>(out, a, b, n_inst, tb.tw, ws);
  } else {
    using C = NttCfg<LOGN, kPolyNttTT>;
    constexpr size_t smem = PolyNttCfg<LOGN>::SMEM_WORDS * sizeof(uint32_t);
    poly_ntt_kernel<LOGN><<<grid, C::T, smem, st>>>(out, a, b, n_inst, tb.tw, ws);
  }
  return cudaGetLastError();
}

template <int LOGN>
static cudaError_t launch_dbg_t(uint32_t* x, uint64_t n_inst, int prime, const NttTables& tb,
                                cudaStream_t st) {
  using C = NttCfg<LOGN>;
  constexpr size_t smem = (size_t)C::XW * sizeof(uint32_t);
  cudaError_t e = cudaFuncSetAttribute(ntt_forward_debug_kernel<LOGN>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  const unsigned grid = cap_grid((unsigned)(n_groups < 65535 ? n_groups : 65535));
  ntt_forward_debug_kernel<LOGN><<<grid, C::T, smem, st>>>(x, n_inst, tb.tw, prime);
  return cudaGetLastError();
}

// 16- or 32-element kernel by size (only the chosen one is instantiated)
template <int LOGN>
static cudaError_t launch_ntt_any_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                   const NttTables& tb, cudaStream_t st, int n_sm) {
  if constexpr (LOGN >= BN_NTT_R32_MIN) return launch_ntt_r32_t<LOGN>(out, a, b, n_inst, tb, st, n_sm);
  else return launch_ntt_t<LOGN>(out, a, b, n_inst, tb, st, n_sm);
}

cudaError_t launch_mul_ntt(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b,
                           uint64_t n_inst, const NttTables& tb, cudaStream_t st, int n_sm) {
  switch (logm + 1) {
#ifdef BN_NTT14_CLUSTER
    case 14: return launch_ntt_cluster_t<14, 512>(out, a, b, n_inst, tb, st, n_sm);
#endif
#ifndef BN_NTT_CL16
    // 32 elements per thread (A/B: 2^19 9.55 -> 8.30 ms, 2^20 12.1 -> 11.5 ms)
    case 15: return launch_ntt_cluster32_t<15>(out, a, b, n_inst, tb, st);
    case 16: return launch_ntt_cluster32_t<16>(out, a, b, n_inst, tb, st);
#else
    case 15: return launch_ntt_cluster_t<15, BN_NTT_CL_T>(out, a, b, n_inst, tb, st, n_sm);
    case 16: return launch_ntt_cluster_t<16, BN_NTT_CL_T>(out, a, b, n_inst, tb, st, n_sm);
#endif
    case 6: return launch_ntt_t<6>(out, a, b, n_inst, tb, st, n_sm);
    case 7: return launch_ntt_t<7>(out, a, b, n_inst, tb, st, n_sm);
    case 8: return launch_ntt_t<8>(out, a, b, n_inst, tb, st, n_sm);
    case 9: return launch_ntt_t<9>(out, a, b, n_inst, tb, st, n_sm);
    case 10: return launch_ntt_t<10>(out, a, b, n_inst, tb, st, n_sm);
    case 11: return launch_ntt_any_t<11>(out, a, b, n_inst, tb, st, n_sm);
    case 12: return launch_ntt_any_t<12>(out, a, b, n_inst, tb, st, n_sm);
    case 13: return launch_ntt_any_t<13>(out, a, b, n_inst, tb, st, n_sm);
#ifndef BN_NTT14_CLUSTER
    case 14: return launch_ntt_any_t<14>(out, a, b, n_inst, tb, st, n_sm);
#endif
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ntt_forward_debug(int lgn, uint32_t* x, uint64_t n_inst, int prime, const NttTables& tb,
                                     cudaStream_t st) {
  switch (lgn) {
    case 6: return launch_dbg_t<6>(x, n_inst, prime, tb, st);
    case 7: return launch_dbg_t<7>(x, n_inst, prime, tb, st);
    case 8: return launch_dbg_t<8>(x, n_inst, prime, tb, st);
    case 9: return launch_dbg_t<9>(x, n_inst, prime, tb, st);
    case 10: return launch_dbg_t<10>(x, n_inst, prime, tb, st);
    case 11: return launch_dbg_t<11>(x, n_inst, prime, tb, st);
    case 12: return launch_dbg_t<12>(x, n_inst, prime, tb, st);
    case 13: return launch_dbg_t<13>(x, n_inst, prime, tb, st);
    case 14: return launch_dbg_t<14>(x, n_inst, prime, tb, st);
    default: return cudaErrorInvalidValue;
  }
}

#define BN_LOGN_SWITCH(F, ...)            \
  switch (logm + 1) {                     \
    case 6: return F<6>(__VA_ARGS__);     \
    case 7: return F<7>(__VA_ARGS__);     \
    case 8: return F<8>(__VA_ARGS__);     \
    case 9: return F<9>(__VA_ARGS__);     \
    case 10: return F<10>(__VA_ARGS__);   \
    case 11: return F<11>(__VA_ARGS__);   \
    case 12: return F<12>(__VA_ARGS__);   \
    case 13: return F<13>(__VA_ARGS__);   \
    case 14: return F<14>(__VA_ARGS__);   \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_mul_wide_ntt(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b,
                                uint64_t n_inst, const NttTables& tb, cudaStream_t st, int n_sm) {
  BN_LOGN_SWITCH(launch_wide_ntt_t, out, a, b, n_inst, tb, st, n_sm)
}

cudaError_t poly_ntt_geometry(int logm, uint64_t n_inst, int n_sm, uint64_t* ws_words) {
  unsigned grid = 0;
  BN_LOGN_SWITCH(poly_ntt_geom_t, n_inst, n_sm, &grid, ws_words)
}

cudaError_t launch_poly_ntt(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                            const NttTables& tb, uint32_t* ws, uint64_t ws_words, cudaStream_t st, int n_sm) {
  BN_LOGN_SWITCH(launch_poly_ntt_t, out, a, b, n_inst, tb, ws, ws_words, st, n_sm)
}

}  // namespace bn
