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
#include <cassert>
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "bn_common.cuh"
#include "bn_kernels.h"

namespace cg = cooperative_groups;

// add at 2^19 / 2^20 bits (A/B on B200, ms per paper batch; 512K / 1M):
//   0: 1024-thread clusters of 2 / 4 CTAs, 8 limbs, cp.async staging, 1 CTA/SM: 0.402 / 0.490
//   1: one CTA x 16 limbs (512K); 2-CTA cluster x 16 limbs, direct loads (1M): 0.331 / 0.379
//   2: clusters of 2 / 4 CTAs, 8 limbs, direct loads, 32 registers, 2 CTAs/SM: 0.310 / 0.336

namespace bn {

template <int LOGM, int L, int BMIN = 256>
struct AddCfg {
  static constexpr int M = 1 << LOGM;
  static constexpr int TPI = M / L;
  static constexpr int BLOCK = TPI > BMIN ? TPI : BMIN;
  static constexpr int IPB = BLOCK / TPI;
};

template <int LOGM, int L>
__global__ void __launch_bounds__(AddCfg<LOGM, L>::BLOCK)
    add_kernel(uint32_t* out, const uint32_t* a,
               const uint32_t* b, uint64_t n_inst) {
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
template <int LOGM, int L, int BMIN>
__global__ void __launch_bounds__(AddCfg<LOGM, L, BMIN>::BLOCK)
    add6_kernel(uint32_t* out, const uint32_t* a,
                const uint32_t* b, uint64_t n_inst) {
  using C = AddCfg<LOGM, L, BMIN>;
  __shared__ uint32_t agg[2][C::BLOCK / 32];
  const uint32_t slot = threadIdx.x / C::TPI;
  const uint32_t lt = threadIdx.x % C::TPI;
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
    uint32_t g, p, cin;
    chunk_sum<L>(x, y, r, g, p);  // a + b
    if (!valid) g = p = 0;
    cin = carry_scan<C::TPI>(g, p, agg[0]);
    add_pending<L, C::TPI>(r, x, cin, p, valid, agg[1]);  // + a
    add_pending<L, C::TPI>(r, y, cin, p, valid, agg[0]);  // + b
    add_pending<L, C::TPI>(r, x, cin, p, valid, agg[1]);  // + a
    add_pending<L, C::TPI>(r, y, cin, p, valid, agg[0]);  // + b
    add_pending<L, C::TPI>(r, x, cin, p, valid, agg[1]);  // + a
    chunk_apply<L>(x, r, cin);
    if (valid) store_limbs<L>(out + off, r);
    if constexpr (C::TPI > 32) __syncthreads();
  }
}

// ------------------------------------------------- 6-Add with a TMA prefetch
// From 64K bits (BN_ADD6_TMA_MIN) the register-resident add6_kernel leaves
// HBM idle: registers (a, b, r: 3 words per limb) hold only two 256K (four
// 128K) instances per SM, each CTA loads its instance, then runs six
// dependent CTA scans, and the loads of all CTAs bunch up (ncu r02 at 256K:
// 35% of the stall samples in load + first scan, long scoreboard).  Here
// every CTA is persistent and owns ONE instance-sized shared stage (a | b,
// 2 m words, 64 KiB at 256K): thread 0 fills it with two tensor bulk copies
// (cp.async.bulk.tensor.2d; the operands viewed as [rows][32 words], one box
// = one instance, 128-byte swizzle so the 16-limbs-per-thread reads are
// bank-conflict free) completing on an mbarrier; the threads copy their
// limbs into registers, and as soon as the first addition's CTA scan has
// passed its barrier (every thread has read the stage) thread 0 refills the
// stage with the CTA's NEXT instance, which then lands while the remaining
// five scans and the store of this one run.  The round-1/2 one-CTA-per-SM
// ring (three stages, re-reading a, b from shared memory) serialised the six
// scans at 0.41 ms; here the residency stays register-bound (2 / 4 / 8 CTAs
// per SM at 256K / 128K / 64K) and only the loads move off the critical path.

// 128-byte swizzle of a TMA box (1024-byte aligned): 16-byte chunk c of row r
// sits at chunk c ^ (r & 7).  Thread lt's 16 limbs are half of row lt / 2,
// chunks 4 (lt & 1) .. +3: the 8 lanes of a quarter-warp then hit 8
// distinct chunks of 4 different rows — conflict free.
// With L = 32 a thread owns row lt (chunks 0..7): again 8 distinct chunks
// per quarter-warp step.
template <int L>
BN_DEV void lds_swz128(uint32_t (&x)[L], const uint32_t* stage, int lt) {
  static_assert(L == 16 || L == 32, "16 or 32 limbs per thread");
  const int row = L == 16 ? lt >> 1 : lt, c0 = L == 16 ? (lt & 1) * 4 : 0;
#pragma unroll
  for (int v = 0; v < L / 4; v++) {
    const uint4 t = *reinterpret_cast<const uint4*>(stage + row * 32 + 4 * ((c0 + v) ^ (row & 7)));
    x[4 * v] = t.x;
    x[4 * v + 1] = t.y;
    x[4 * v + 2] = t.z;
    x[4 * v + 3] = t.w;
  }
}

template <int LOGM>
struct Add6TmaCfg {
  static constexpr int M = 1 << LOGM, L = LOGM >= BN_ADD6_TMA_L32 ? 32 : 16, T = M / L, ROWS = M / 32;
  static constexpr int MINB = (L == 32 ? 512 : 1024) / T;  // 128 / 64 registers
  static constexpr size_t SMEM = 2 * (size_t)M * 4 + 1024;  // a | b stage + alignment slack
  static_assert(ROWS <= 256, "one TMA box per operand (box rows <= 256)");
  static_assert(T >= 64, "the first scan must contain a CTA barrier");
};

template <int LOGM>
__global__ void __launch_bounds__(Add6TmaCfg<LOGM>::T, Add6TmaCfg<LOGM>::MINB)
    add6_tma_kernel(uint32_t* out, const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b, uint64_t n_inst) {
  using C = Add6TmaCfg<LOGM>;
  constexpr int M = C::M, L = C::L, T = C::T;
  extern __shared__ uint8_t smem_raw[];
  // align by an offset from the shared array itself (not by integer casts of
  // a generic pointer), so the stage reads stay LDS.128, not generic LD
  const uint32_t pad = (1024u - (mbar_addr(smem_raw) & 1023u)) & 1023u;
  uint32_t* As = reinterpret_cast<uint32_t*>(smem_raw + pad);
  uint32_t* Bs = As + M;
  __shared__ __align__(8) uint64_t full;
  __shared__ uint32_t agg[2][T / 32];
  const int lt = threadIdx.x;
#ifdef BN_BOUNDS_CHECK  // debug builds (scripts/bounds_check.sh): the aligned stage fits the allocation
  assert(pad + 2u * M * 4u <= C::SMEM && (mbar_addr(As) & 1023u) == 0 && blockDim.x == T);
  assert((L == 16 ? lt >> 1 : lt) < M / 32);
#endif
  auto issue = [&](uint64_t inst) {  // thread 0
    mbar_expect_tx(&full, 2 * M * 4);
    tma_load_2d(As, &map_a, 0, (int)(inst * C::ROWS), &full);
    tma_load_2d(Bs, &map_b, 0, (int)(inst * C::ROWS), &full);
  };
  if (lt == 0) {
    mbar_init(&full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (lt == 0 && blockIdx.x < n_inst) issue(blockIdx.x);
  uint32_t phase = 0;
  for (uint64_t inst = blockIdx.x; inst < n_inst; inst += gridDim.x, phase ^= 1) {
    mbar_wait(&full, phase);
    uint32_t x[L], y[L], r[L];
    lds_swz128<L>(x, As, lt);
    lds_swz128<L>(y, Bs, lt);
    uint32_t g, p, cin;
    chunk_sum<L>(x, y, r, g, p);  // a + b
    cin = carry_scan<T>(g, p, agg[0]);
    // carry_scan's CTA barrier: every thread has read the stage -> refill it
    if (lt == 0 && inst + gridDim.x < n_inst) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(inst + gridDim.x);
    }
    add_pending<L, T>(r, x, cin, p, true, agg[1]);  // + a
    add_pending<L, T>(r, y, cin, p, true, agg[0]);  // + b
    add_pending<L, T>(r, x, cin, p, true, agg[1]);  // + a
    add_pending<L, T>(r, y, cin, p, true, agg[0]);  // + b
    add_pending<L, T>(r, x, cin, p, true, agg[1]);  // + a
    chunk_apply<L>(x, r, cin);
    store_limbs<L>(out + inst * (uint64_t)M + lt * L, r);
    // the next instance's first scan writes agg[0]: its last readers (the
    // fifth scan) are ordered before the sixth scan's barrier
  }
}

// host: a [rows][32 words] view of one operand (rows = n_inst * m / 32), box
// 32 words x m / 32 rows (one instance), 128-byte swizzle
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess) return nullptr;
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}
static cudaError_t add6_tensor_map(CUtensorMap* map, const uint32_t* base, uint64_t rows, uint32_t box_rows) {
  // driver entry point, resolved once (thread-safe static initialisation)
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  if (!encode) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {32, rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {32, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(base), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int LOGM>
static cudaError_t launch_add6_tma_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                     cudaStream_t st, int n_sm) {
  using C = Add6TmaCfg<LOGM>;
  const uint64_t rows = n_inst * (uint64_t)C::M / 32;
  if (rows >= (1ull << 31)) return cudaErrorInvalidValue;  // TMA coordinates are int32
  CUtensorMap ma, mb;
  cudaError_t e = add6_tensor_map(&ma, a, rows, C::ROWS);
  if (e != cudaSuccess) return e;
  e = add6_tensor_map(&mb, b, rows, C::ROWS);
  if (e != cudaSuccess) return e;
  static LaunchCache cache;
  int per_sm = 0;
  e = resident_ctas(cache, add6_tma_kernel<LOGM>, C::T, C::SMEM, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t cap = (uint64_t)n_sm * per_sm;  // persistent: one resident wave
  const unsigned grid = cap_grid((unsigned)(n_inst < cap ? n_inst : cap));
  add6_tma_kernel<LOGM><<<grid, C::T, C::SMEM, st>>>(out, ma, mb, n_inst);
  return cudaGetLastError();
}

// Sizes beyond one CTA (2^19, 2^20 bits): one instance per
// thread-block cluster of CR = M / (1024 L) CTAs, CTA rank r holding
// limbs [r M/CR, (r+1) M/CR), 1024 threads x L limbs.  The carry scan runs
// across the cluster (cluster_carry_scan: the CTA aggregates travel through
// DSMEM) — the hierarchical scan of PAPER.md:289-292 with one more level,
// instead of the single-pass decoupled look-back over global memory the
// paper cites.
// NS > 0: each thread stages the next NS - 1 instances' 2 x L limbs into
// shared memory with cp.async (NS stages of 64 KiB per CTA) while it scans
// and stores the current one; a thread only ever reads back what it copied
// itself (no CTA barrier needed).  NS = 0: limbs are loaded straight into
// registers, and with MB = 2 (32 registers) two clusters share each SM so
// one's loads overlap the other's cluster barrier — the default (BN_ADD_BIG).
template <int LOGM, int L, int NS, int MB>
__global__ void __launch_bounds__(1024, MB)
    add_cluster_kernel(uint32_t* out, const uint32_t* a,
                       const uint32_t* b, uint64_t n_inst) {
  constexpr int M = 1 << LOGM, CR = M / (1024 * L), SL = M / CR;  // limbs per CTA
  extern __shared__ __align__(16) uint32_t sm[];  // [NS stages][a | b][SL]
  __shared__ uint32_t agg[32];
  __shared__ uint32_t cta_agg[2 * CR];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const uint64_t n_cl = gridDim.x / CR;
  const uint32_t lo = threadIdx.x * L;
  // every CTA of the cluster must be running before any CTA writes into its
  // shared memory (the first cluster_carry_scan stores into the other CTAs'
  // cta_agg before its own cluster barrier; compute-sanitizer racecheck r02)
  cl.sync();
  auto stage = [&](uint64_t inst, int st) {
    const uint64_t off = inst * (uint64_t)M + (uint64_t)rank * SL + lo;
    uint32_t* s = sm + st * 2 * SL;
#pragma unroll
    for (int v = 0; v < L / 4; v++) {
      cp_async16(s + lo + 4 * v, a + off + 4 * v, true);
      cp_async16(s + SL + lo + 4 * v, b + off + 4 * v, true);
    }
  };
  uint64_t inst = blockIdx.x / CR;
  // prologue: the first NS - 1 instances in flight
#pragma unroll
  for (int k = 0; k < NS - 1; k++) {
    if (inst + k * n_cl < n_inst) stage(inst + k * n_cl, k);
    cp_async_commit();
  }
  int parity = 0;
  for (int st = 0; inst < n_inst; inst += n_cl, parity ^= 1, st = st >= NS - 1 ? 0 : st + 1) {
    uint32_t x[L], y[L], r[L], g, p;
    const uint64_t off = inst * (uint64_t)M + (uint64_t)rank * SL + lo;
    if constexpr (NS > 0) {
      const int sf = st == 0 ? NS - 1 : st - 1;  // stage of instance inst + (NS-1) n_cl
      if (inst + (NS - 1) * n_cl < n_inst) stage(inst + (NS - 1) * n_cl, sf);
      cp_async_commit();
      cp_async_wait<NS - 1>();
      lds_limbs<L>(x, sm + st * 2 * SL + lo);
      lds_limbs<L>(y, sm + st * 2 * SL + SL + lo);
    } else {
      load_limbs<L>(x, a + off);
      load_limbs<L>(y, b + off);
    }
    chunk_sum<L>(x, y, r, g, p);
    const uint32_t cin = cluster_carry_scan<CR>(g, p, agg, cta_agg, parity, cl);
    chunk_apply<L>(x, r, cin);
    store_limbs<L>(out + off, r);
  }
  if constexpr (NS > 0) cp_async_wait<0>();
}

// ------------------------------------------------------------ beyond clusters
// bn_add_big: any power-of-two size from 2^18 to 2^30 bits with the
// single-pass decoupled look-back scan the paper's carry-scan citation refers
// to — the way past what one CTA (2^18) or one
// thread-block cluster (2^20) can hold.  Every instance is cut into tiles of
// 8192 limbs (2^18 bits; 1024 threads x 8 limbs, loaded straight into
// registers); CTAs take tiles in order from an atomic counter, so every
// tile's predecessors have started (no deadlock whatever the scheduling).
// A tile publishes its aggregate (g = carry-out with carry-in 0, p = every
// limb sum all ones) as soon as its CTA scan is done, looks back for its
// carry-in, then publishes its inclusive carry-out.  For the carry operator
// the look-back is short: a predecessor with p = 0 is already decisive
// (carry = g, whatever came into it), only all-ones tiles pass the carry on.
// One warp reads 32 predecessors' flags at once and takes the nearest
// decisive one (an instance's first tile has carry-in 0).  Flag word:
// bits 0-1 status (0 none, 1 aggregate, 2 inclusive), bit 2 g, bit 3 p,
// bit 4 inclusive carry-out; payload and status in one 32-bit store, so no
// fence is needed between them.  Flags and the counter live in a caller
// workspace zeroed (cudaMemsetAsync) before the launch.
constexpr int kLbThreads = BN_ADD_BIG_THREADS, kLbL = 8, kLbTile = kLbThreads * kLbL;  // limbs per tile

BN_DEV uint32_t ld_flag(const uint32_t* f) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}
BN_DEV void st_flag(uint32_t* f, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kLbThreads, 2048 / kLbThreads)
    add_lookback_kernel(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t total_tiles,
                        uint32_t tiles_per_inst, uint32_t* flags, uint32_t* counter) {
  __shared__ uint32_t tile_s, cin_s;
  __shared__ uint32_t agg[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 32) agg[tid] = 2u;  // warps past the CTA's count: the operator's identity (g 0, p 1)
  if (tid == 0) tile_s = atomicAdd(counter, 1u);
  __syncthreads();
  const uint64_t order = tile_s;
  if (order >= total_tiles) return;
  // tiles are taken tile-index-major (tile lt of every instance before tile
  // lt + 1 of any): a tile's predecessor was taken n_inst tiles earlier, so
  // with many instances in flight it has usually published its inclusive
  // carry already and the look-back is one read
  const uint64_t n_inst = total_tiles / tiles_per_inst;
  const uint32_t lt = (uint32_t)(order / n_inst);      // tile index within its instance
  const uint64_t tile = (order % n_inst) * tiles_per_inst + lt;  // instance-major flag / data index
  const uint64_t off = tile * (uint64_t)kLbTile + tid * kLbL;  // instances are contiguous
  uint32_t x[kLbL], y[kLbL], r[kLbL], g, p;
  load_limbs<kLbL>(x, a + off);
  load_limbs<kLbL>(y, b + off);
  chunk_sum<kLbL>(x, y, r, g, p);
  // lane and warp levels (ballot-add), as in carry_scan / cluster_carry_scan
  const uint32_t G = __ballot_sync(0xFFFFFFFFu, g), P = __ballot_sync(0xFFFFFFFFu, p), X = G | P;
  if (lane == 0) agg[warp] = (uint32_t)(((uint64_t)X + G) >> 32) | ((P == 0xFFFFFFFFu) << 1);
  __syncthreads();
  const uint32_t av = agg[lane];
  const uint32_t G2 = __ballot_sync(0xFFFFFFFFu, av & 1u), P2 = __ballot_sync(0xFFFFFFFFu, (av >> 1) & 1u);
  const uint32_t X2 = G2 | P2;
  if (warp == 0) {
    const uint32_t gT = (uint32_t)(((uint64_t)X2 + G2) >> 32), pT = P2 == 0xFFFFFFFFu;
    uint32_t C = 0;
    if (lt == 0) {
      if (lane == 0) st_flag(flags + tile, 2u | (gT << 2) | (pT << 3) | (gT << 4));
    } else {
      if (lane == 0) st_flag(flags + tile, 1u | (gT << 2) | (pT << 3));
      // look back over the instance's earlier tiles, 32 at a time
      uint64_t base = tile;  // window: base-1-lane
      uint32_t remaining = lt;  // earlier tiles of this instance
      for (;;) {
        const bool in = lane < remaining;
        uint32_t f = 0;
        if (in) {
          do {
            f = ld_flag(flags + base - 1 - lane);
          } while ((f & 3u) == 0);
        }
        // decisive: inclusive published, or an aggregate that kills / generates (p = 0);
        // lanes past the instance's first tile count as decisive with carry 0
        const bool dec = !in || (f & 3u) == 2u || !((f >> 3) & 1u);
        const uint32_t dm = __ballot_sync(0xFFFFFFFFu, dec);
        if (dm) {
          const int d = __ffs(dm) - 1;
          const uint32_t fd = __shfl_sync(0xFFFFFFFFu, f, d);
          const bool ind = d < (int)remaining;
          C = !ind ? 0u : ((fd & 3u) == 2u ? (fd >> 4) & 1u : (fd >> 2) & 1u);
          break;
        }
        base -= 32;
        remaining -= 32;
      }
      if (lane == 0) st_flag(flags + tile, 2u | (gT << 2) | (pT << 3) | ((gT | (pT & C)) << 4));
    }
    if (lane == 0) cin_s = C;
  }
  __syncthreads();
  const uint32_t C = cin_s;
  const uint32_t c0 = (((X2 + G2 + C) ^ X2 ^ G2) >> warp) & 1u;
  const uint32_t cin = (((X + G + c0) ^ X ^ G) >> lane) & 1u;
  chunk_apply<kLbL>(x, r, cin);
  store_limbs<kLbL>(out + off, r);
}

uint64_t add_big_workspace_words(int logm, uint64_t n_inst) {
  const uint64_t tiles = n_inst * ((1ull << logm) / kLbTile);
  return (tiles + 1 + 3) & ~3ull;  // flags + counter, 16-byte multiple
}

cudaError_t launch_add_big(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                           uint32_t* ws, uint64_t ws_words, cudaStream_t st) {
  const uint32_t tpi = (uint32_t)((1ull << logm) / kLbTile);
  const uint64_t total = n_inst * tpi;
  if (tpi < 1 || total >= (1ull << 31) || ws_words < add_big_workspace_words(logm, n_inst))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(ws, 0, (total + 1) * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  add_lookback_kernel<<<(unsigned)total, kLbThreads, 0, st>>>(out, a, b, total, tpi, ws + 1, ws);
  return cudaGetLastError();
}

template <int LOGM, int L = 8, int NS = BN_ADD_CL_STAGES, int MB = 1>
static cudaError_t launch_add_cluster_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                        cudaStream_t st, int n_sm) {
  constexpr int CR = (1 << LOGM) / (1024 * L);
  cudaLaunchConfig_t cfg = {};
  constexpr size_t smem = NS * 2 * ((1 << LOGM) / CR) * sizeof(uint32_t);
  cfg.gridDim = dim3(CR);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CR;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent clusters: exactly as many as can be co-resident (clusters must
  // fit in one GPC, so this is below n_sm / CR); more would run as a second
  // wave and double the time
  static LaunchCache cache;
  int max_cl = 0;
  cudaError_t e = cached_query(cache, [&](int* o) {
    cudaError_t e1 = cudaFuncSetAttribute(add_cluster_kernel<LOGM, L, NS, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e1 != cudaSuccess) return e1;
    return cudaOccupancyMaxActiveClusters(o, add_cluster_kernel<LOGM, L, NS, MB>, &cfg);
  }, &max_cl);
  if (e != cudaSuccess) return e;
  if (max_cl < 1) return cudaErrorInvalidConfiguration;
  uint64_t n_cl = n_inst < (uint64_t)max_cl ? n_inst : (uint64_t)max_cl;
  n_cl = cap_grid((unsigned)n_cl);
  cfg.gridDim = dim3((unsigned)(n_cl * CR));
  e = cudaLaunchKernelEx(&cfg, add_cluster_kernel<LOGM, L, NS, MB>, out, a, b, n_inst);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// 6-Add geometry (A/B on one box, ms per paper batch).  Limbs per thread:
// L = 8 up to 8K bits (one warp per instance); 16K: L = 16 (TPI = 32, no
// CTA barrier: 0.335 -> 0.264 ms); 32K: L = 8 (16: 0.386, 32: 0.445);
// 64K, 128K, 256K: L = 16 (L = 8 at 256K: 40 registers x 1024 threads left
// one CTA per SM, 0.555 -> 0.377 ms; L = 32: 128K 0.341 -> 0.474).  CTAs
// from 32K bits hold one instance (BLOCK = TPI >= 128 instead of >= 256):
// 32K 0.324 -> 0.286, 64K 0.320 -> 0.296.  Parking a and b in shared memory
// (32 registers) and a cp.async double-buffered persistent variant both
// measured slower (256K 0.435 / 0.586 ms).
constexpr int add6_limbs_per_thread(int logm) {
  return logm <= 8 ? 8 : logm == 9 ? 16 : logm == 10 ? 8 : logm == 11 ? 16 : logm == 12 ? BN_ADD6_L12 : BN_ADD6_L13;
}

template <int LOGM>
static cudaError_t launch_add6_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                 cudaStream_t st, int n_sm) {
  constexpr int L = add6_limbs_per_thread(LOGM);
  constexpr int BMIN = LOGM >= 10 ? BN_ADD6_BMIN_MID : 256;
  using C = AddCfg<LOGM, L, BMIN>;
  const uint64_t n_groups = (n_inst + C::IPB - 1) / C::IPB;
  const uint64_t per_sm = 2048 / C::BLOCK;
  const uint64_t cap = (uint64_t)n_sm * per_sm * 8;
  const unsigned grid = cap_grid((unsigned)(n_groups < cap ? n_groups : cap));
  add6_kernel<LOGM, L, BMIN><<<grid, C::BLOCK, 0, st>>>(out, a, b, n_inst);
  return cudaGetLastError();
}

template <int LOGM, int L = 8>
static cudaError_t launch_add_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                cudaStream_t st, int n_sm) {
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
    // 2^19 on one CTA (1024 threads x 16 limbs, 38 registers): 0.402 ms
    // (2-CTA cluster, 8 limbs) -> 0.329 ms by A/B; 2^20 on a 2-CTA cluster
    // with 16 limbs per thread, loaded straight into registers
#if BN_ADD_BIG == 1
    case 14: return launch_add_t<14, 16>(out, a, b, n_inst, st, n_sm);
    case 15: return launch_add_cluster_t<15, 16, 0>(out, a, b, n_inst, st, n_sm);
#elif BN_ADD_BIG == 2
    case 14: return launch_add_cluster_t<14, 8, 0, 2>(out, a, b, n_inst, st, n_sm);
    case 15: return launch_add_cluster_t<15, 8, 0, 2>(out, a, b, n_inst, st, n_sm);
#else
    case 14: return launch_add_cluster_t<14>(out, a, b, n_inst, st, n_sm);
    case 15: return launch_add_cluster_t<15>(out, a, b, n_inst, st, n_sm);
#endif
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
  if (logm >= BN_ADD6_TMA_MIN) {
    switch (logm) {
      case 10: return launch_add6_tma_t<10>(out, a, b, n_inst, st, n_sm);
      case 11: return launch_add6_tma_t<11>(out, a, b, n_inst, st, n_sm);
      case 12: return launch_add6_tma_t<12>(out, a, b, n_inst, st, n_sm);
      case 13: return launch_add6_tma_t<13>(out, a, b, n_inst, st, n_sm);
      default: break;
    }
  }
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
