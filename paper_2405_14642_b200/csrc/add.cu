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

// ------------------------------------------------------------ 6-Add fed by TMA
// From 32K bits (BN_ADD6_TMA_MIN) the register-resident add6_kernel exposes
// its load latency: ncu r02 at 256K puts 35% of the stall samples in the
// load + first-scan phase (long-scoreboard 55% of them), and registers (a, b
// and r: 3 words per limb) cap the SM at two 256K instances, so HBM idles
// while the six dependent CTA scans run (0.66 - 0.77 of the copy bandwidth at
// 128K / 256K).  Here one persistent 512-thread CTA per SM streams its
// instances through a 3-stage ring in shared memory: thread 0 issues two
// tensor bulk copies per stage (cp.async.bulk.tensor.2d — the operands as a
// [rows][32 words] tensor, 256 rows = 32 KiB per operand per stage, 128-byte
// swizzle so the 16-limbs-per-thread reads are bank-conflict free) that
// complete on the stage's mbarrier; the threads wait on it, run the six
// carry-save additions with only r in registers (a and b are re-read from
// the stage, four limbs at a time) and store r.  The last scan's CTA barrier
// orders every read of a stage before thread 0 refills it, so two stages
// (64 KiB each) are always in flight while one is consumed.
constexpr int kA6Threads = 512;                 // per CTA
constexpr int kA6Rows = kA6Threads * 16 / 32;   // 256 rows of 32 words per operand per stage
constexpr int kA6StageBytes = 2 * kA6Rows * 128;  // a | b
constexpr int kA6Stages = 3;

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
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(mbar_addr(dst)), "l"(map), "r"(c0), "r"(c1), "r"(mbar_addr(bar))
      : "memory");
}

// 128-byte swizzle of the TMA box: 16-byte chunk c of row r sits at chunk
// c ^ (r & 7) (the smem stage is 1024-byte aligned).
BN_DEV const uint4* a6_chunk(const uint32_t* stage, int row, int c) {
  return reinterpret_cast<const uint4*>(stage + row * 32 + 4 * (c ^ (row & 7)));
}

template <int L, bool BOTH>
BN_DEV void chunk_sum_tma(uint32_t (&r)[L], const uint32_t* xs, const uint32_t* ys, int row, int c0,
                          uint32_t cin, uint32_t& g, uint32_t& p) {
  uint32_t c = cin, all = 0xFFFFFFFFu;
#pragma unroll
  for (int v = 0; v < L / 4; v++) {
    const uint4 yv = *a6_chunk(ys, row, c0 + v);
    uint32_t xv[4];
    if constexpr (BOTH) {
      const uint4 t = *a6_chunk(xs, row, c0 + v);
      xv[0] = t.x; xv[1] = t.y; xv[2] = t.z; xv[3] = t.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; i++) xv[i] = r[4 * v + i];
    }
    const uint32_t yy[4] = {yv.x, yv.y, yv.z, yv.w};
    uint32_t t[4];
    c = add4_cc(t, xv, yy, c);
#pragma unroll
    for (int i = 0; i < 4; i++) {
      r[4 * v + i] = t[i];
      all &= t[i];
    }
  }
  g = c;
  p = all == 0xFFFFFFFFu;
}

template <int LOGM>
__global__ void __launch_bounds__(kA6Threads, 1)
    add6_tma_kernel(uint32_t* out, const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b, uint64_t n_inst) {
  constexpr int L = 16, M = 1 << LOGM, TPI = M / L, IPB = kA6Threads / TPI;
  static_assert(TPI >= 64 && TPI <= kA6Threads, "32K .. 256K bits");
  extern __shared__ uint8_t smem_raw[];
  uint32_t* ring = reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kA6Stages];
  __shared__ uint32_t agg[2][kA6Threads / 32];
  const int tid = threadIdx.x;
  const int slot = tid / TPI, lt = tid % TPI;
  const uint64_t n_items = (n_inst + IPB - 1) / IPB;
  auto issue = [&](uint64_t item, int s) {
    uint32_t* st = ring + s * (kA6StageBytes / 4);
    mbar_expect_tx(&full[s], kA6StageBytes);
    const int row0 = (int)(item * kA6Rows);  // rows of 32 words: item * IPB * M / 32
    tma_load_2d(st, &map_a, 0, row0, &full[s]);
    tma_load_2d(st + kA6Rows * 32, &map_b, 0, row0, &full[s]);
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kA6Stages; s++) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kA6Stages; s++) {
      const uint64_t item = blockIdx.x + (uint64_t)s * gridDim.x;
      if (item < n_items) issue(item, s);
    }
  }
  // this thread's 16 limbs: row (slot M + 16 lt) / 32 of the stage, chunks c0 .. c0+3
  const int row = (slot * M + lt * L) / 32;
  const int c0 = ((lt * L) % 32) / 4;
  int s = 0;
  uint32_t phase = 0;
  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint32_t* st = ring + s * (kA6StageBytes / 4);
    const uint32_t* as = st;
    const uint32_t* bs = st + kA6Rows * 32;
    mbar_wait(&full[s], phase);
    const uint64_t inst = item * IPB + slot;
    const bool valid = inst < n_inst;
    uint32_t r[L], g, p, cin;
    chunk_sum_tma<L, true>(r, as, bs, row, c0, 0u, g, p);  // a + b
    if (!valid) g = p = 0;
    cin = carry_scan<TPI>(g, p, agg[0]);
#pragma unroll
    for (int k = 1; k < 6; k++) {  // + a, + b, + a, + b, + a  (carry-save, as add_pending)
      const uint32_t ov = p & cin;
      chunk_sum_tma<L, false>(r, nullptr, (k & 1) ? as : bs, row, c0, cin, g, p);
      g &= ~ov;
      if (!valid) g = p = 0;
      cin = carry_scan<TPI>(g, p, agg[k & 1]);
    }
    // the last scan's CTA barrier: every thread is done reading this stage
    if (tid == 0) {
      const uint64_t nxt = item + (uint64_t)kA6Stages * gridDim.x;
      if (nxt < n_items) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(nxt, s);
      }
    }
    chunk_apply<L>(r, r, cin);
    if (valid) store_limbs<L>(out + inst * (uint64_t)M + lt * L, r);
    __syncthreads();  // agg[0] reused by the next item's first scan
    if (++s == kA6Stages) {
      s = 0;
      phase ^= 1;
    }
  }
}

// host: a [rows][32 words] view of one operand (rows = n_inst * M / 32), box
// 32 words x kA6Rows rows, 128-byte swizzle
static cudaError_t a6_tensor_map(CUtensorMap* map, const uint32_t* base, uint64_t rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {32, rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {32, (cuuint32_t)kA6Rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(base), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int LOGM>
static cudaError_t launch_add6_tma_t(uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                                     cudaStream_t st, int n_sm) {
  constexpr int M = 1 << LOGM, IPB = kA6Threads / (M / 16);
  constexpr size_t smem = (size_t)kA6Stages * kA6StageBytes + 1024;
  const uint64_t rows = n_inst * (uint64_t)M / 32;
  if (rows >= (1ull << 31)) return cudaErrorInvalidValue;  // TMA coordinates are int32
  CUtensorMap ma, mb;
  cudaError_t e = a6_tensor_map(&ma, a, rows);
  if (e != cudaSuccess) return e;
  e = a6_tensor_map(&mb, b, rows);
  if (e != cudaSuccess) return e;
  static LaunchCache cache;
  int per_sm = 0;
  e = resident_ctas(cache, add6_tma_kernel<LOGM>, kA6Threads, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t n_items = (n_inst + IPB - 1) / IPB;
  const uint64_t cap = (uint64_t)n_sm * per_sm;
  const unsigned grid = cap_grid((unsigned)(n_items < cap ? n_items : cap));
  add6_tma_kernel<LOGM><<<grid, kA6Threads, smem, st>>>(out, ma, mb, n_inst);
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
