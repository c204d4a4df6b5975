// bn_api.cu — the C ABI of libbn.so (include/bn.h): argument validation,
// size -> kernel dispatch, per-device NTT constant tables, and the pipelined
// host-buffer entry point.  Host code only; kernels live in add.cu,
// mul_classical.cu and mul_ntt.cu.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/bn.h"
#include "bn_config.h"
#include "bn_kernels.h"

namespace bn {
unsigned g_grid_cap = 0;
}

namespace {

thread_local int tls_cuda_err = 0;

constexpr int kMaxDev = 64;
constexpr uint32_t kMinBits = 1024, kMaxBits = 1048576;
// bn_add_big: 2^18 .. 2^30 bits (tiles of 2^18 bits, decoupled look-back)
constexpr int kBigMinLb = 18, kBigMaxLb = 30;

// Largest log2(bits) per operation: 2^18 fits one CTA (the paper's range);
// add and the NTT product go to 2^20, the classical product to 2^19, on
// thread-block clusters; the fused and wide products stop
// at 2^18.
int op_max_lb(int op) {
  switch (op) {
    case BN_OP_ADD: case BN_OP_MUL_NTT: return 20;
    case BN_OP_MUL_CLASSICAL: return 19;
    case BN_OP_ADD6: case BN_OP_POLY_CLASSICAL: case BN_OP_POLY_NTT: case BN_OP_MUL_WIDE_CLASSICAL:
    case BN_OP_MUL_WIDE_NTT: return 18;
    default: return -1;
  }
}

// The three NTT primes, p0 < p1 < p2 < 2^30, each p = k 2^17 + 1 (the three
// largest such primes below 2^30, so every N = 2^6 .. 2^17 has a primitive
// N-th root), product 2^89.99 > 2^79 >= the largest coefficient
// m (2^32-1)^2 at m = 32768 (1M-bit operands, reading R10).
// Verified prime at start-up by a deterministic Miller-Rabin.
constexpr uint32_t kPrimes[bn::kNumPrimes] = {1070727169u, 1071513601u, 1073479681u};

// ---------------------------------------------------------------- number theory (host)
uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((unsigned __int128)a * b % m); }
uint64_t powmod(uint64_t a, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  a %= m;
  while (e) {
    if (e & 1) r = mulmod(r, a, m);
    a = mulmod(a, a, m);
    e >>= 1;
  }
  return r;
}
bool is_prime_u32(uint32_t n) {
  if (n < 2) return false;
  for (uint32_t q : {2u, 3u, 5u, 7u}) {
    if (n % q == 0) return n == q;
  }
  uint32_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) { d >>= 1; s++; }
  for (uint32_t a : {2u, 3u, 5u, 7u}) {  // deterministic for n < 3.2e9
    uint64_t x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; r++) {
      x = mulmod(x, x, n);
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}
uint32_t inv_mod(uint32_t a, uint32_t p) { return (uint32_t)powmod(a, p - 2, p); }
uint32_t shoup_of(uint32_t w, uint32_t p) { return (uint32_t)(((uint64_t)w << 32) / p); }
uint32_t primitive_root(uint32_t p) {
  std::vector<uint32_t> fs;
  uint32_t n = p - 1;
  for (uint32_t q = 2; (uint64_t)q * q <= n; q++) {
    if (n % q == 0) {
      fs.push_back(q);
      while (n % q == 0) n /= q;
    }
  }
  if (n > 1) fs.push_back(n);
  for (uint32_t g = 2;; g++) {
    bool ok = true;
    for (uint32_t q : fs)
      if (powmod(g, (p - 1) / q, p) == 1) { ok = false; break; }
    if (ok) return g;
  }
}

// ---------------------------------------------------------------- per-device state
struct DevState {
  // set (release) once the tables are uploaded; read (acquire) without the lock
  std::atomic<bool> ready{false};
  int n_sm = 0;
  uint2* tw_dev = nullptr;
  bn::NttTables tables[bn::kMaxLogN + 1];
  // bn_run_host scratch
  cudaStream_t st[BN_RUN_HOST_STREAMS] = {};
  uint32_t* scratch = nullptr;
  size_t scratch_bytes = 0;
};
DevState g_dev[kMaxDev];
std::mutex g_mu;
bool g_consts_ok = false;
bn::PrimeConst g_pc[bn::kNumPrimes];

bn_status cuda_fail(cudaError_t e) {
  tls_cuda_err = (int)e;
  return BN_ECUDA;
}

bool host_consts() {
  if (g_consts_ok) return true;
  for (int j = 0; j < bn::kNumPrimes; j++) {
    const uint32_t p = kPrimes[j];
    if (!is_prime_u32(p) || ((p - 1) & ((1u << bn::kMaxLogN) - 1)) != 0 || p >= (1u << 30)) return false;
    uint32_t inv = p;  // Newton: p^-1 mod 2^32
    for (int i = 0; i < 5; i++) inv *= 2u - p * inv;
    g_pc[j] = {p, 2 * p, (uint32_t)(0u - inv), shoup_of(1, p)};
  }
  g_consts_ok = true;
  return true;
}

// tables for every N = 2^6 .. 2^14 on the current device
bn_status build_tables(DevState& d) {
  size_t total = 0;
  for (int lg = bn::kMinLogN; lg <= bn::kMaxLogN; lg++) total += (size_t)bn::kNumPrimes * 2 * ((1u << lg) - 1);
  std::vector<uint2> host(total);
  size_t off = 0;
  bn::CrtConst crt[bn::kMaxLogN + 1];
  std::memset(crt, 0, sizeof(crt));
  const uint32_t p0 = kPrimes[0], p1 = kPrimes[1], p2 = kPrimes[2];
  size_t lg_off[bn::kMaxLogN + 1] = {0};
  for (int lg = bn::kMinLogN; lg <= bn::kMaxLogN; lg++) {
    const uint32_t N = 1u << lg;
    bn::NttTables& tb = d.tables[lg];
    lg_off[lg] = off;
    for (int j = 0; j < bn::kNumPrimes; j++) {
      const uint32_t p = kPrimes[j];
      const uint32_t g = primitive_root(p);
      const uint32_t w = (uint32_t)powmod(g, (p - 1) / N, p);
      tb.omega[j] = w;
      for (int dir = 0; dir < 2; dir++) {
        const uint32_t base = dir == 0 ? w : inv_mod(w, p);
        for (int s = 0; s < lg; s++) {
          const uint32_t step = (uint32_t)powmod(base, 1ull << s, p);
          uint32_t cur = 1;
          const uint32_t cnt = N >> (s + 1);
          uint2* T = host.data() + off + (N - (N >> s));
          for (uint32_t k = 0; k < cnt; k++) {
            T[k] = make_uint2(cur, shoup_of(cur, p));
            cur = (uint32_t)mulmod(cur, step, p);
          }
        }
        off += N - 1;
      }
    }
    // CRT constants folded with K_j = 2^32 N^-1 mod p_j
    uint32_t K[3];
    for (int j = 0; j < 3; j++) {
      const uint32_t p = kPrimes[j];
      K[j] = (uint32_t)mulmod(powmod(2, 32, p), inv_mod(N % p, p), p);
    }
    bn::CrtConst c;
    const uint32_t i01 = inv_mod(p0 % p1, p1);
    const uint64_t p01 = (uint64_t)p0 * p1;
    const uint32_t i012 = inv_mod((uint32_t)(p01 % p2), p2);
    c.k0 = K[0];
    c.k0_sh = shoup_of(c.k0, p0);
    c.k1i = (uint32_t)mulmod(K[1], i01, p1);
    c.k1i_sh = shoup_of(c.k1i, p1);
    c.i01 = i01;
    c.i01_sh = shoup_of(i01, p1);
    c.k2i = (uint32_t)mulmod(K[2], i012, p2);
    c.k2i_sh = shoup_of(c.k2i, p2);
    c.i012 = i012;
    c.i012_sh = shoup_of(i012, p2);
    c.p0i012 = (uint32_t)mulmod(p0 % p2, i012, p2);
    c.p0i012_sh = shoup_of(c.p0i012, p2);
    c.p01_lo = (uint32_t)p01;
    c.p01_hi = (uint32_t)(p01 >> 32);
    crt[lg] = c;
  }
  cudaError_t e = cudaMalloc(&d.tw_dev, total * sizeof(uint2));
  if (e != cudaSuccess) return cuda_fail(e);
  e = cudaMemcpy(d.tw_dev, host.data(), total * sizeof(uint2), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e);
  for (int lg = bn::kMinLogN; lg <= bn::kMaxLogN; lg++) d.tables[lg].tw = d.tw_dev + lg_off[lg];
  e = bn::upload_prime_consts(g_pc, crt);
  if (e != cudaSuccess) return cuda_fail(e);
  return BN_OK;
}

bn_status ensure_device(int dev, DevState** out) {
  if (dev < 0 || dev >= kMaxDev) return BN_ENODEV;
  DevState& d = g_dev[dev];
  if (d.ready.load(std::memory_order_acquire)) {
    *out = &d;
    return BN_OK;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  if (!d.ready.load(std::memory_order_relaxed)) {
    if (!host_consts()) return BN_EINVAL;
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) return cuda_fail(e);
    // the library holds sm_100a code only: any other compute capability
    // (10.x with x != 0, 12.x, ...) cannot load it
    if (prop.major != 10 || prop.minor != 0) return BN_ENODEV;
    d.n_sm = prop.multiProcessorCount;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
    bn_status st = build_tables(d);
    if (prev != dev) cudaSetDevice(prev);
    if (st != BN_OK) return st;
    d.ready.store(true, std::memory_order_release);
  }
  *out = &d;
  return BN_OK;
}

bn_status current_device(DevState** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  return ensure_device(dev, out);
}

int ilog2_exact(uint64_t v) {
  if (v == 0 || (v & (v - 1))) return -1;
  int r = 0;
  while ((1ull << r) < v) r++;
  return r;
}

// validation shared by the three ops; returns log2(u32 limbs)
bn_status validate(int op, const void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                   uint32_t limb_bits, int* logm) {
  if (limb_bits != 32 && limb_bits != 64) return BN_EINVAL;
  if (n_limbs == 0) return BN_EINVAL;
  const uint64_t bits = (uint64_t)n_limbs * limb_bits;
  const int lb = ilog2_exact(bits);
  if (lb < 10 || lb > op_max_lb(op)) return BN_ESIZE;
  *logm = lb - 5;
  if (n_inst == 0) return BN_OK;
  if (!out || !a || !b) return BN_EINVAL;
  if (((uintptr_t)out | (uintptr_t)a | (uintptr_t)b) & 15) return BN_EALIGN;
  const uint64_t bytes = n_inst * (bits / 8);
  auto overl = [&](const void* x, const void* y) {
    const uintptr_t x0 = (uintptr_t)x, y0 = (uintptr_t)y;
    return x0 != y0 && x0 < y0 + bytes && y0 < x0 + bytes;
  };
  if (overl(out, a) || overl(out, b)) return BN_EALIAS;
  return BN_OK;
}

bn_status run_op(int op, void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                 uint32_t limb_bits, cudaStream_t st) {
  int logm = 0;
  bn_status s = validate(op, out, a, b, n_inst, n_limbs, limb_bits, &logm);
  if (s != BN_OK || n_inst == 0) return s;
  DevState* d = nullptr;
  s = current_device(&d);
  if (s != BN_OK) return s;
  cudaError_t e;
  uint32_t* o = (uint32_t*)out;
  const uint32_t* x = (const uint32_t*)a;
  const uint32_t* y = (const uint32_t*)b;
  switch (op) {
    case BN_OP_ADD: e = bn::launch_add(logm, o, x, y, n_inst, st, d->n_sm); break;
    case BN_OP_MUL_CLASSICAL: e = bn::launch_mul_classical(logm, o, x, y, n_inst, st, d->n_sm); break;
    case BN_OP_MUL_NTT: e = bn::launch_mul_ntt(logm, o, x, y, n_inst, d->tables[logm + 1], st, d->n_sm); break;
    case BN_OP_ADD6: e = bn::launch_add6(logm, o, x, y, n_inst, st, d->n_sm); break;
    default: return BN_EINVAL;
  }
  return e == cudaSuccess ? BN_OK : cuda_fail(e);
}

// Full products: out holds 2 n_limbs limbs per instance (partial overlap with
// an input is rejected; out may not equal an input either, it is twice as large)
bn_status run_wide(int op, void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                   uint32_t limb_bits, cudaStream_t st) {
  int logm = 0;
  // operand checks (out is checked below against its doubled size)
  bn_status s = validate(op, a, a, a, n_inst, n_limbs, limb_bits, &logm);
  if (s != BN_OK) return s;
  if (n_inst && !b) return BN_EINVAL;
  if (n_inst && ((uintptr_t)b & 15)) return BN_EALIGN;
  if (n_inst == 0) return BN_OK;
  if (!out) return BN_EINVAL;
  if ((uintptr_t)out & 15) return BN_EALIGN;
  const uint64_t bytes = n_inst * ((uint64_t)n_limbs * limb_bits / 8);
  auto overl = [](const void* x, uint64_t xn, const void* y, uint64_t yn) {
    const uintptr_t x0 = (uintptr_t)x, y0 = (uintptr_t)y;
    return x0 < y0 + yn && y0 < x0 + xn;
  };
  if (overl(out, 2 * bytes, a, bytes) || overl(out, 2 * bytes, b, bytes)) return BN_EALIAS;
  DevState* d = nullptr;
  s = current_device(&d);
  if (s != BN_OK) return s;
  cudaError_t e = op == BN_OP_MUL_WIDE_CLASSICAL
                      ? bn::launch_mul_wide_classical(logm, (uint32_t*)out, (const uint32_t*)a,
                                                      (const uint32_t*)b, n_inst, st, d->n_sm)
                      : bn::launch_mul_wide_ntt(logm, (uint32_t*)out, (const uint32_t*)a, (const uint32_t*)b,
                                                n_inst, d->tables[logm + 1], st, d->n_sm);
  return e == cudaSuccess ? BN_OK : cuda_fail(e);
}

bool is_poly(int op) { return op == BN_OP_POLY_CLASSICAL || op == BN_OP_POLY_NTT; }

// workspace words of a Poly call (one slice per resident CTA of its grid)
bn_status poly_ws_words(int op, int logm, uint64_t n_inst, const DevState* d, uint64_t* words) {
  cudaError_t e = op == BN_OP_POLY_CLASSICAL ? bn::poly_classical_geometry(logm, n_inst, d->n_sm, words)
                                             : bn::poly_ntt_geometry(logm, n_inst, d->n_sm, words);
  return e == cudaSuccess ? BN_OK : cuda_fail(e);
}

bn_status launch_poly(int op, int logm, uint32_t* o, const uint32_t* x, const uint32_t* y, uint64_t n_inst,
                      uint32_t* ws, uint64_t ws_words, cudaStream_t st, const DevState* d) {
  cudaError_t e = op == BN_OP_POLY_CLASSICAL
                      ? bn::launch_poly_classical(logm, o, x, y, n_inst, ws, ws_words, st, d->n_sm)
                      : bn::launch_poly_ntt(logm, o, x, y, n_inst, d->tables[logm + 1], ws, ws_words, st, d->n_sm);
  return e == cudaSuccess ? BN_OK : cuda_fail(e);
}

bn_status run_poly(int op, void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                   uint32_t limb_bits, void* ws, uint64_t ws_bytes, cudaStream_t st) {
  int logm = 0;
  bn_status s = validate(op, out, a, b, n_inst, n_limbs, limb_bits, &logm);
  if (s != BN_OK || n_inst == 0) return s;
  DevState* d = nullptr;
  s = current_device(&d);
  if (s != BN_OK) return s;
  uint64_t need = 0;
  s = poly_ws_words(op, logm, n_inst, d, &need);
  if (s != BN_OK) return s;
  if (!ws || ((uintptr_t)ws & 15)) return ws ? BN_EALIGN : BN_EINVAL;
  if (ws_bytes < need * 4) return BN_EINVAL;
  const uint64_t bytes = n_inst * ((uint64_t)n_limbs * limb_bits / 8);
  auto overl = [](const void* x, uint64_t xn, const void* y, uint64_t yn) {
    const uintptr_t x0 = (uintptr_t)x, y0 = (uintptr_t)y;
    return x0 < y0 + yn && y0 < x0 + xn;
  };
  if (overl(ws, need * 4, out, bytes) || overl(ws, need * 4, a, bytes) || overl(ws, need * 4, b, bytes))
    return BN_EALIAS;
  return launch_poly(op, logm, (uint32_t*)out, (const uint32_t*)a, (const uint32_t*)b, n_inst, (uint32_t*)ws,
                     need, st, d);
}

}  // namespace

extern "C" {

bn_status bn_add(void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                 uint32_t limb_bits, bn_stream_t stream) {
  return run_op(BN_OP_ADD, out, a, b, n_inst, n_limbs, limb_bits, (cudaStream_t)stream);
}

bn_status bn_mul_classical(void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                           uint32_t limb_bits, bn_stream_t stream) {
  return run_op(BN_OP_MUL_CLASSICAL, out, a, b, n_inst, n_limbs, limb_bits, (cudaStream_t)stream);
}

bn_status bn_mul_ntt(void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                     uint32_t limb_bits, bn_stream_t stream) {
  return run_op(BN_OP_MUL_NTT, out, a, b, n_inst, n_limbs, limb_bits, (cudaStream_t)stream);
}

bn_status bn_add6(void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs, uint32_t limb_bits,
                  bn_stream_t stream) {
  return run_op(BN_OP_ADD6, out, a, b, n_inst, n_limbs, limb_bits, (cudaStream_t)stream);
}

bn_status bn_mul_wide_classical(void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                                 uint32_t limb_bits, bn_stream_t stream) {
  return run_wide(BN_OP_MUL_WIDE_CLASSICAL, out, a, b, n_inst, n_limbs, limb_bits, (cudaStream_t)stream);
}

bn_status bn_mul_wide_ntt(void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                          uint32_t limb_bits, bn_stream_t stream) {
  return run_wide(BN_OP_MUL_WIDE_NTT, out, a, b, n_inst, n_limbs, limb_bits, (cudaStream_t)stream);
}

uint64_t bn_poly_workspace_bytes(int op, uint64_t n_inst, uint32_t n_limbs, uint32_t limb_bits) {
  if (!is_poly(op)) return 0;
  int logm = 0;
  if (validate(op, (void*)16, (void*)16, (void*)16, 0, n_limbs, limb_bits, &logm) != BN_OK) return 0;
  if (n_inst == 0) return 0;
  DevState* d = nullptr;
  if (current_device(&d) != BN_OK) return 0;
  uint64_t w = 0;
  if (poly_ws_words(op, logm, n_inst, d, &w) != BN_OK) return 0;
  return w * 4;
}

bn_status bn_poly_classical(void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                            uint32_t limb_bits, void* workspace, uint64_t workspace_bytes, bn_stream_t stream) {
  return run_poly(BN_OP_POLY_CLASSICAL, out, a, b, n_inst, n_limbs, limb_bits, workspace, workspace_bytes,
                  (cudaStream_t)stream);
}

bn_status bn_poly_ntt(void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs,
                      uint32_t limb_bits, void* workspace, uint64_t workspace_bytes, bn_stream_t stream) {
  return run_poly(BN_OP_POLY_NTT, out, a, b, n_inst, n_limbs, limb_bits, workspace, workspace_bytes,
                  (cudaStream_t)stream);
}

uint64_t bn_add_big_workspace_bytes(uint64_t n_inst, uint32_t n_limbs, uint32_t limb_bits) {
  if (limb_bits != 32 && limb_bits != 64) return 0;
  const int lb = ilog2_exact((uint64_t)n_limbs * limb_bits);
  if (lb < kBigMinLb || lb > kBigMaxLb || n_inst == 0) return 0;
  return bn::add_big_workspace_words(lb - 5, n_inst) * 4;
}

bn_status bn_add_big(void* out, const void* a, const void* b, uint64_t n_inst, uint32_t n_limbs, uint32_t limb_bits,
                     void* workspace, uint64_t workspace_bytes, bn_stream_t stream) {
  if (limb_bits != 32 && limb_bits != 64) return BN_EINVAL;
  if (n_limbs == 0) return BN_EINVAL;
  const uint64_t bits = (uint64_t)n_limbs * limb_bits;
  const int lb = ilog2_exact(bits);
  if (lb < kBigMinLb || lb > kBigMaxLb) return BN_ESIZE;
  if (n_inst == 0) return BN_OK;
  if (!out || !a || !b || !workspace) return BN_EINVAL;
  if (((uintptr_t)out | (uintptr_t)a | (uintptr_t)b | (uintptr_t)workspace) & 15) return BN_EALIGN;
  const uint64_t bytes = n_inst * (bits / 8);
  const uint64_t need = bn::add_big_workspace_words(lb - 5, n_inst) * 4;
  if (need / 4 >= (1ull << 31)) return BN_ESIZE;  // one CTA per tile: the grid is an int32
  if (workspace_bytes < need) return BN_EINVAL;
  auto overl = [](const void* x, uint64_t xn, const void* y, uint64_t yn) {
    const uintptr_t x0 = (uintptr_t)x, y0 = (uintptr_t)y;
    return x0 < y0 + yn && y0 < x0 + xn;
  };
  auto partial = [&](const void* x, const void* y) { return x != y && overl(x, bytes, y, bytes); };
  if (partial(out, a) || partial(out, b)) return BN_EALIAS;
  if (overl(workspace, need, out, bytes) || overl(workspace, need, a, bytes) || overl(workspace, need, b, bytes))
    return BN_EALIAS;
  DevState* d = nullptr;
  bn_status s = current_device(&d);
  if (s != BN_OK) return s;
  cudaError_t e = bn::launch_add_big(lb - 5, (uint32_t*)out, (const uint32_t*)a, (const uint32_t*)b, n_inst,
                                     (uint32_t*)workspace, need / 4, (cudaStream_t)stream);
  return e == cudaSuccess ? BN_OK : cuda_fail(e);
}

bn_status bn_prepare(int device) {
  DevState* d = nullptr;
  return ensure_device(device, &d);
}

bn_status bn_run_host(const int* ops, void* const* outs, int n_ops, const void* a, const void* b,
                      uint64_t n_inst, uint32_t n_limbs, uint32_t limb_bits) {
  if (n_ops <= 0 || !ops || !outs) return BN_EINVAL;
  int logm = 0;
  // validate sizes with dummy aligned device pointers (host buffers may alias-check only)
  for (int i = 0; i < n_ops; i++) {
    if (ops[i] < BN_OP_ADD || ops[i] > BN_OP_POLY_NTT) return BN_EINVAL;
    bn_status s = validate(ops[i], (void*)16, (void*)16, (void*)16, 0, n_limbs, limb_bits, &logm);
    if (s != BN_OK) return s;
  }
  if (n_inst == 0) return BN_OK;
  if (!a || !b) return BN_EINVAL;
  for (int i = 0; i < n_ops; i++)
    if (!outs[i]) return BN_EINVAL;
  bn_status s;
  DevState* d = nullptr;
  s = current_device(&d);
  if (s != BN_OK) return s;
  const size_t inst_bytes = (size_t)4 << logm;
  // chunk: ~BN_RUN_HOST_CHUNK_MB MiB per operand, at least one instance
  uint64_t chunk = ((uint64_t)BN_RUN_HOST_CHUNK_MB << 20) / inst_bytes;
  if (chunk < 1) chunk = 1;
  if (chunk > n_inst) chunk = n_inst;
  const size_t chunk_bytes = chunk * inst_bytes;
  // Poly workspace per stream (the largest of the two methods' needs for one chunk)
  uint64_t ws_words = 0;
  for (int i = 0; i < n_ops; i++) {
    if (!is_poly(ops[i])) continue;
    uint64_t w = 0;
    s = poly_ws_words(ops[i], logm, chunk, d, &w);
    if (s != BN_OK) return s;
    if (w > ws_words) ws_words = w;
  }
  const size_t ws_bytes = ((size_t)ws_words * 4 + 255) & ~(size_t)255;
  const size_t per_stream = chunk_bytes * (2 + (size_t)n_ops) + ws_bytes;
  std::lock_guard<std::mutex> lk(g_mu);  // scratch is per device, one pipeline at a time
  cudaError_t e;
  constexpr int NS = BN_RUN_HOST_STREAMS;
  if (!d->st[NS - 1]) {  // all or none: a partial failure leaves no null stream behind
    for (int i = 0; i < NS; i++) {
      if (d->st[i]) continue;
      e = cudaStreamCreateWithFlags(&d->st[i], cudaStreamNonBlocking);
      if (e != cudaSuccess) {
        d->st[i] = nullptr;
        return cuda_fail(e);
      }
    }
  }
  if (d->scratch_bytes < NS * per_stream) {
    if (d->scratch) cudaFree(d->scratch);
    d->scratch = nullptr;
    d->scratch_bytes = 0;
    e = cudaMalloc(&d->scratch, NS * per_stream);
    if (e != cudaSuccess) return cuda_fail(e);
    d->scratch_bytes = NS * per_stream;
  }
  const char* ha = (const char*)a;
  const char* hb = (const char*)b;
  // on any failure, drain both streams before returning: copies and kernels
  // of earlier chunks must not keep writing into the caller's host buffers
  // (or reading this scratch) after the call has returned
  auto fail = [&](bn_status st) {
    for (int i = 0; i < NS; i++) (void)cudaStreamSynchronize(d->st[i]);
    return st;
  };
  auto fail_cuda = [&](cudaError_t err) {
    const bn_status st = cuda_fail(err);
    return fail(st);
  };
  uint64_t c = 0;
  for (uint64_t i0 = 0; i0 < n_inst; i0 += chunk, c++) {
    const uint64_t n = (n_inst - i0) < chunk ? (n_inst - i0) : chunk;
    const size_t bytes = n * inst_bytes;
    cudaStream_t st = d->st[c % NS];
    char* base = (char*)d->scratch + (c % NS) * per_stream;
    uint32_t* da = (uint32_t*)base;
    uint32_t* db = (uint32_t*)(base + chunk_bytes);
    e = cudaMemcpyAsync(da, ha + i0 * inst_bytes, bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail_cuda(e);
    e = cudaMemcpyAsync(db, hb + i0 * inst_bytes, bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail_cuda(e);
    for (int k = 0; k < n_ops; k++) {
      uint32_t* dout = (uint32_t*)(base + (2 + k) * chunk_bytes);
      uint32_t* dws = (uint32_t*)(base + (2 + n_ops) * chunk_bytes);
      switch (ops[k]) {
        case BN_OP_ADD: e = bn::launch_add(logm, dout, da, db, n, st, d->n_sm); break;
        case BN_OP_MUL_CLASSICAL: e = bn::launch_mul_classical(logm, dout, da, db, n, st, d->n_sm); break;
        case BN_OP_MUL_NTT: e = bn::launch_mul_ntt(logm, dout, da, db, n, d->tables[logm + 1], st, d->n_sm); break;
        case BN_OP_ADD6: e = bn::launch_add6(logm, dout, da, db, n, st, d->n_sm); break;
        default: {
          s = launch_poly(ops[k], logm, dout, da, db, n, dws, ws_words, st, d);
          if (s != BN_OK) return fail(s);
          e = cudaSuccess;
        }
      }
      if (e != cudaSuccess) return fail_cuda(e);
      e = cudaMemcpyAsync((char*)outs[k] + i0 * inst_bytes, dout, bytes, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return fail_cuda(e);
    }
  }
  for (int i = 0; i < NS; i++) {
    e = cudaStreamSynchronize(d->st[i]);
    if (e != cudaSuccess) return fail_cuda(e);
  }
  return BN_OK;
}

uint32_t bn_max_bits(void) { return kMaxBits; }
uint32_t bn_min_bits(void) { return kMinBits; }
int bn_cuda_error(void) { return tls_cuda_err; }

const char* bn_status_string(bn_status s) {
  switch (s) {
    case BN_OK: return "BN_OK";
    case BN_EINVAL: return "BN_EINVAL: invalid argument";
    case BN_ESIZE: return "BN_ESIZE: bits must be a power of two in [1024, bn_op_max_bits(op)]";
    case BN_EALIGN: return "BN_EALIGN: buffers must be 16-byte aligned";
    case BN_EALIAS: return "BN_EALIAS: out partially overlaps an input";
    case BN_ECUDA: return "BN_ECUDA: CUDA error (see bn_cuda_error)";
    case BN_ENODEV: return "BN_ENODEV: no usable sm_100 device";
  }
  return "unknown bn_status";
}

uint32_t bn_op_max_bits(int op) {
  const int lb = op_max_lb(op);
  return lb < 0 ? 0u : (1u << lb);
}

uint32_t bn_launches_per_call(int op, uint32_t bits) {
  const int lb = ilog2_exact(bits);
  if (lb < 10 || lb > op_max_lb(op)) return 0;
  return 1;
}

void bn_debug_set_grid_cap(uint32_t cap) { bn::g_grid_cap = cap; }

void bn_ntt_primes(uint32_t p[3]) {
  for (int j = 0; j < 3; j++) p[j] = kPrimes[j];
}

bn_status bn_debug_ntt_forward(uint32_t* x, uint64_t n_inst, uint32_t lg_n, int prime, uint32_t* omega_out,
                               bn_stream_t stream) {
  if ((int)lg_n < bn::kMinLogN || (int)lg_n > bn::kMaxLogNOneCta || prime < 0 || prime >= bn::kNumPrimes)
    return BN_EINVAL;
  DevState* d = nullptr;
  bn_status s = current_device(&d);
  if (s != BN_OK) return s;
  if (omega_out) *omega_out = d->tables[lg_n].omega[prime];
  if (n_inst == 0) return BN_OK;
  if (!x) return BN_EINVAL;
  cudaError_t e = bn::launch_ntt_forward_debug((int)lg_n, x, n_inst, prime, d->tables[lg_n], (cudaStream_t)stream);
  return e == cudaSuccess ? BN_OK : cuda_fail(e);
}

}  // extern "C"
