// add.cu — bn_add: batched fixed-width addition as a carry-propagation scan.
//
// PAPER.md:144-163 (§2): (1) map p_i = a_i + b_i with (ov_i, mx_i),
// (2) exclusive scan of the carry pairs, (3) map r_i = p_i + carry_i;
// batched as bbadd, with efficient sequentialization
// (PAPER.md:283-327): each thread owns L = 8 consecutive u32 limbs held in
// registers, loaded and stored with 128-bit streaming accesses straight
// from/to HBM — shared memory is used only for the (<= 32-word) warp
// aggregates of the CTA-level scan.
//
// Work map: m = 2^LOGM limbs per instance, TPI = m / L threads per instance
// (4 at 1K bits ... 1024 at 256K bits).  A CTA of BLOCK = max(256, TPI)
// threads handles IPB = BLOCK / TPI instances; the grid is persistent-ish
// (grid-stride over instance groups) so small sizes amortise launch and
// tail effects.  HBM-bound: 3 * bits / 8 algorithmic bytes per instance
// (PAPER.md:929).
#include "bn_common.cuh"
#include "bn_kernels.h"

namespace bn {

template <int LOGM, int L>
struct AddCfg {
  static constexpr int M = 1 << LOGM;
  static constexpr int TPI = M / L;
  static constexpr int BLOCK = TPI > 256 ? TPI : 256;
  static constexpr int IPB = BLOCK / TPI;
};

template <int LOGM, int L>
__global__ void __launch_bounds__(AddCfg<LOGM, L>::BLOCK)
    add_kernel(uint32_t* __restrict__ out, const uint32_t* __restrict__ a,
               const uint32_t* __restrict__ b, uint64_t n_inst) {
  using C = AddCfg<LOGM, L>;
  __shared__ uint32_t agg[C::BLOCK / 32];
  const uint32_t slot = threadIdx.x / C::TPI;  // instance slot in the CTA
  const uint32_t lt = threadIdx.x % C::TPI;    // thread within the instance
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  for (uint64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const uint64_t inst = grp * C::IPB + slot;
    const bool valid = inst < n_inst;
    const uint64_t off = inst * (uint64_t)C::M + (uint64_t)lt * L;
    uint32_t x[L], y[L], r[L];
    if (valid) {
      load_limbs<L>(x, a + off);
      load_limbs<L>(y, b + off);
    } else {
#pragma unroll
      for (int i = 0; i < L; i++) x[i] = y[i] = 0;
    }
    add_regs<L, C::TPI>(x, y, r, valid, agg);
    if (valid) store_limbs<L>(out + off, r);
    if constexpr (C::TPI > 32) __syncthreads();  // agg reused next iteration
  }
}

// 6-Add (Table 1): six dependent additions fused in one
// kernel with every intermediate held in registers (block-level fusion).
// The paper does not print the expression; reading R17:
// r = a + b, then alternately + a, + b, i.e. r = 4a + 3b mod 2^bits — six
// full carry scans, each one the §2 map -> scan -> map.  The two agg
// buffers alternate so consecutive scans need no extra barrier (a scan's
// own __syncthreads orders every thread's previous read of the other buffer).
template <int LOGM, int L>
__global__ void __launch_bounds__(AddCfg<LOGM, L>::BLOCK)
    add6_kernel(uint32_t* __restrict__ out, const uint32_t* __restrict__ a,
                const uint32_t* __restrict__ b, uint64_t n_inst) {
  using C = AddCfg<LOGM, L>;
  __shared__ uint32_t agg[2][C::BLOCK / 32];
  const uint32_t slot = threadIdx.x / C::TPI;
  const uint32_t lt = threadIdx.x % C::TPI;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  for (uint64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const uint64_t inst = grp * C::IPB + slot;
    const bool valid = inst < n_inst;
    const uint64_t off = inst * (uint64_t)C::M + (uint64_t)lt * L;
    uint32_t x[L], y[L], r[L], s[L];
    if (valid) {
      load_limbs<L>(x, a + off);
      load_limbs<L>(y, b + off);
    } else {
#pragma unroll
      for (int i = 0; i < L; i++) x[i] = y[i] = 0;
    }
    add_regs<L, C::TPI>(x, y, r, valid, agg[0]);  // a + b
    add_regs<L, C::TPI>(r, x, s, valid, agg[1]);  // + a
    add_regs<L, C::TPI>(s, y, r, valid, agg[0]);  // + b
    add_regs<L, C::TPI>(r, x, s, valid, agg[1]);  // + a
    add_regs<L, C::TPI>(s, y, r, valid, agg[0]);  // + b
    add_regs<L, C::TPI>(r, x, s, valid, agg[1]);  // + a
    if (valid) store_limbs<L>(out + off, s);
    if constexpr (C::TPI > 32) __syncthreads();
  }
}

template <int LOGM>
static cudaError_t launch_add6_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                 cudaStream_t st, int n_sm) {
  constexpr int L = 8;
  using C = AddCfg<LOGM, L>;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  const uint64_t per_sm = 2048 / C::BLOCK;
  const uint64_t cap = (uint64_t)n_sm * per_sm * 8;
  const unsigned grid = cap_grid((unsigned)(n_groups < cap ? n_groups : cap));
  add6_kernel<LOGM, L><<<grid, C::BLOCK, 0, st>>>(out, a, b, n_inst);
  return cudaGetLastError();
}

template <int LOGM>
static cudaError_t launch_add_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                cudaStream_t st, int n_sm) {
  constexpr int L = 8;
  using C = AddCfg<LOGM, L>;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  // resident CTAs per SM for this block size (2048 threads/SM)
  const uint64_t per_sm = 2048 / C::BLOCK;
  const uint64_t cap = (uint64_t)n_sm * per_sm * 8;  // several waves of work per CTA slot
  const unsigned grid = cap_grid((unsigned)(n_groups < cap ? n_groups : cap));
  add_kernel<LOGM, L><<<grid, C::BLOCK, 0, st>>>(out, a, b, n_inst);
  return cudaGetLastError();
}

cudaError_t launch_add(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                       cudaStream_t st, int n_sm) {
  switch (logm) {
    case 5: return launch_add_t<5>(out, a, b, n_inst, st, n_sm);
    case 6: return launch_add_t<6>(out, a, b, n_inst, st, n_sm);
    case 7: return launch_add_t<7>(out, a, b, n_inst, st, n_sm);
    case 8: return launch_add_t<8>(out, a, b, n_inst, st, n_sm);
    case 9: return launch_add_t<9>(out, a, b, n_inst, st, n_sm);
    case 10: return launch_add_t<10>(out, a, b, n_inst, st, n_sm);
    case 11: return launch_add_t<11>(out, a, b, n_inst, st, n_sm);
    case 12: return launch_add_t<12>(out, a, b, n_inst, st, n_sm);
    case 13: return launch_add_t<13>(out, a, b, n_inst, st, n_sm);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_add6(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                        cudaStream_t st, int n_sm) {
  switch (logm) {
    case 5: return launch_add6_t<5>(out, a, b, n_inst, st, n_sm);
    case 6: return launch_add6_t<6>(out, a, b, n_inst, st, n_sm);
    case 7: return launch_add6_t<7>(out, a, b, n_inst, st, n_sm);
    case 8: return launch_add6_t<8>(out, a, b, n_inst, st, n_sm);
    case 9: return launch_add6_t<9>(out, a, b, n_inst, st, n_sm);
    case 10: return launch_add6_t<10>(out, a, b, n_inst, st, n_sm);
    case 11: return launch_add6_t<11>(out, a, b, n_inst, st, n_sm);
    case 12: return launch_add6_t<12>(out, a, b, n_inst, st, n_sm);
    case 13: return launch_add6_t<13>(out, a, b, n_inst, st, n_sm);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bn
