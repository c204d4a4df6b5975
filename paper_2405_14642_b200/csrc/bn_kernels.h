// bn_kernels.h — internal interface between the host dispatcher (bn_api.cu)
// and the kernel translation units.  Not part of the public C ABI.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace bn {

constexpr int kNumPrimes = 3;
constexpr int kMinLogN = 6;   // N = 2m, m = 32 limbs (1024 bits)
constexpr int kMaxLogN = 16;  // m = 32768 limbs (1048576 bits; N > 2^14 runs on a CTA cluster)
constexpr int kMaxLogNOneCta = 14;  // m = 8192 limbs (262144 bits): one instance per CTA

// Per-prime constants of the exact NTT product (host-computed in bn_api.cu).
struct PrimeConst {
  uint32_t p;      // prime, 2^29 < p < 2^30, p = k 2^17 + 1
  uint32_t p2;     // 2p
  uint32_t pinv;   // -p^-1 mod 2^32 (Montgomery)
  uint32_t one_sh; // floor(2^32 / p): Shoup constant of w = 1 (input reduction)
};

// Garner CRT constants (p0 < p1 < p2), folded with the inverse-transform
// normalisation K_j = 2^32 * N^-1 mod p_j (Montgomery R and 1/N).  Each
// multiplier is a Shoup pair (w, floor(w 2^32 / p)).
struct CrtConst {
  uint32_t k0, k0_sh;          // mod p0: K0
  uint32_t k1i, k1i_sh;        // mod p1: K1 * p0^-1
  uint32_t i01, i01_sh;        // mod p1: p0^-1
  uint32_t k2i, k2i_sh;        // mod p2: K2 * (p0 p1)^-1
  uint32_t i012, i012_sh;      // mod p2: (p0 p1)^-1
  uint32_t p0i012, p0i012_sh;  // mod p2: p0 (p0 p1)^-1
  uint32_t p01_lo, p01_hi;     // p0 * p1 (< 2^60)
};

// Twiddle tables for one transform length N = 2^lg, contiguous: the table of
// prime j and direction d (0 = forward omega, 1 = inverse omega^-1) starts at
// tw + (2 j + d) (N - 1); inside it stage s occupies entries
// [N - (N >> s), N - (N >> (s+1))) holding (w^(k 2^s), Shoup(w^(k 2^s))) for
// k < N >> (s+1).
struct NttTables {
  const uint2* tw;
  uint32_t omega[kNumPrimes];  // primitive N-th roots used (host side; debug/tests)
};

// Per-device cache of a launch-geometry query (cudaFuncSetAttribute for the
// dynamic shared memory + an occupancy query): microseconds per call on the
// host, and the answer never changes for a (kernel instantiation, device).
// One static LaunchCache per call site; 0 = not yet known.
struct LaunchCache {
  std::atomic<int> v[64];
};
template <class Query>
inline cudaError_t cached_query(LaunchCache& c, Query&& q, int* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const bool ok = dev >= 0 && dev < 64;
  if (ok) {
    const int v = c.v[dev].load(std::memory_order_relaxed);
    if (v > 0) {
      *out = v;
      return cudaSuccess;
    }
  }
  e = q(out);
  if (e == cudaSuccess && ok && *out > 0) c.v[dev].store(*out, std::memory_order_relaxed);
  return e;
}
// resident CTAs per SM of `kernel` with `threads` threads and `smem` bytes of
// dynamic shared memory (sets the opt-in shared-memory limit on first use)
template <class K>
inline cudaError_t resident_ctas(LaunchCache& c, K kernel, int threads, size_t smem, int* per_sm) {
  return cached_query(c, [&](int* o) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(o, kernel, threads, smem);
  }, per_sm);
}

// prime constants + per-lg CRT constants -> __constant__ memory of the current device
// Test knob (bn_debug_set_grid_cap): when > 0, every launcher caps its grid
// at this many CTAs, forcing the grid-stride / persistent paths on small batches.
extern unsigned g_grid_cap;
inline unsigned cap_grid(unsigned g) { return (g_grid_cap && g > g_grid_cap) ? g_grid_cap : g; }

cudaError_t upload_prime_consts(const PrimeConst (&pc)[kNumPrimes], const CrtConst (&crt)[kMaxLogN + 1]);

cudaError_t launch_add(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                       cudaStream_t st, int n_sm);
cudaError_t launch_mul_classical(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b,
                                 uint64_t n_inst, cudaStream_t st, int n_sm);
cudaError_t launch_mul_ntt(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b,
                           uint64_t n_inst, const NttTables& tb, cudaStream_t st, int n_sm);
// add beyond the cluster sizes (decoupled look-back over 8192-limb tiles),
// logm 13 .. 25; the workspace (flags + tile counter) is zeroed per launch
uint64_t add_big_workspace_words(int logm, uint64_t n_inst);
cudaError_t launch_add_big(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                           uint32_t* ws, uint64_t ws_words, cudaStream_t st);
// Fused workloads: 6-Add and Poly.  The Poly kernels use
// a caller-provided workspace of ws_words u32 words, sized by *_geometry for
// the same (logm, n_inst, n_sm) — one slice per resident CTA.
cudaError_t launch_add6(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                        cudaStream_t st, int n_sm);
cudaError_t poly_classical_geometry(int logm, uint64_t n_inst, int n_sm, uint64_t* ws_words);
cudaError_t launch_poly_classical(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b,
                                  uint64_t n_inst, uint32_t* ws, uint64_t ws_words, cudaStream_t st,
                                  int n_sm);
cudaError_t poly_ntt_geometry(int logm, uint64_t n_inst, int n_sm, uint64_t* ws_words);
cudaError_t launch_poly_ntt(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b, uint64_t n_inst,
                            const NttTables& tb, uint32_t* ws, uint64_t ws_words, cudaStream_t st, int n_sm);
// Full (untruncated) products: out has 2^(logm+1) u32 limbs per instance.
// Both support logm <= 13 (inputs up to 256K bits).
cudaError_t launch_mul_wide_classical(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b,
                                      uint64_t n_inst, cudaStream_t st, int n_sm);
cudaError_t launch_mul_wide_ntt(int logm, uint32_t* out, const uint32_t* a, const uint32_t* b,
                                uint64_t n_inst, const NttTables& tb, cudaStream_t st, int n_sm);
cudaError_t launch_ntt_forward_debug(int lgn, uint32_t* x, uint64_t n_inst, int prime,
                                     const NttTables& tb, cudaStream_t st);

}  // namespace bn
