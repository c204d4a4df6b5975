// int_peak.cu — integer-pipe throughput microbenchmark for sm_100a.
//
// Measures sustained warp-instruction throughput (lanes per SM clock) for the
// integer instruction classes the hot path is built from (SURVEY.md §8(d),
// "measure with int_peak"): IMAD (mad.lo), IMAD.HI (mul.hi), IMAD.WIDE.U32
// (mad.wide), the column mad-chain PP (mad.lo.cc/madc.hi.cc/addc), IADD3,
// LOP3, VIMNMX (min.u32), and an IMAD+IADD3 mix that shows dual-pipe issue.
//
// Each thread runs ILP independent chains; cycles are taken from clock64()
// per CTA (SM clock domain), so the result is in lanes/clk/SM, independent of
// the (variable) SM frequency.  Wall time via CUDA events gives ops/s at the
// clock the part actually ran.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak int_peak.cu
// Output: one JSON object per op on stdout.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int ILP = 8;
constexpr int ITERS = 4096;

enum Op { IMAD_LO, IMAD_HI, IMAD_WIDE, MADCHAIN, IADD3_, LOP3_, VMIN_, MIX_IMAD_IADD, NOPS };
static const char* op_name[NOPS] = {"imad_lo", "imad_hi", "imad_wide", "madchain_pp",
                                    "iadd3", "lop3", "vimnmx", "mix_imad_iadd3"};
// SASS instructions per "op" unit, for reporting instr/clk as well
static const double op_instr[NOPS] = {1, 1, 1, 1.5, 1, 1, 1, 2};

template <int OP>
__global__ void kern(uint32_t* out, uint32_t seed, long long* cyc) {
  uint32_t r[ILP], s[ILP], t[ILP];
#pragma unroll
  for (int k = 0; k < ILP; k++) { r[k] = seed + threadIdx.x * 7 + k; s[k] = seed ^ (k * 0x9e3779b9u); t[k] = k; }
  uint32_t a = seed * 3 + 1, b = seed * 5 + 7;
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int k = 0; k < ILP; k++) {
      if (OP == IMAD_LO) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[k]) : "r"(a), "r"(s[k]));
      if (OP == IMAD_HI) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(r[k]) : "r"(a));
      if (OP == IMAD_WIDE) {
        uint64_t w; asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(r[k]), "r"(a), "l"(((uint64_t)s[k] << 32) | r[k]));
        r[k] = (uint32_t)w; s[k] = (uint32_t)(w >> 32);
      }
      if (OP == MADCHAIN)
        asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
                     : "+r"(r[k]), "+r"(s[k]), "+r"(t[k]) : "r"(a + k), "r"(b));
      if (OP == IADD3_) asm volatile("add.u32 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
      if (OP == LOP3_) asm volatile("xor.b32 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
      if (OP == VMIN_) asm volatile("min.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(r[k]) : "r"(s[k]), "r"(a));
      if (OP == MIX_IMAD_IADD) asm volatile("mad.lo.u32 %0, %0, %2, %1;\n\tadd.u32 %1, %1, %3;" : "+r"(r[k]), "+r"(s[k]) : "r"(a), "r"(b));
    }
  }
  long long c1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < ILP; k++) acc ^= r[k] ^ s[k] ^ t[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

template <int OP>
int run(int nsm, int ctas_per_sm, int threads) {
  int grid = nsm * ctas_per_sm;
  uint32_t* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(uint32_t) * grid * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * grid));
  kern<OP><<<grid, threads>>>(out, 1, cyc);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<OP><<<grid, threads>>>(out, 2, cyc);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* hc = new long long[grid];
  CK(cudaMemcpy(hc, cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost));
  long long cmax = 0; double cavg = 0;
  for (int i = 0; i < grid; i++) { if (hc[i] > cmax) cmax = hc[i]; cavg += hc[i]; }
  cavg /= grid;
  // ops issued per SM (all resident CTAs run concurrently by construction)
  double units = (double)ctas_per_sm * threads * ITERS * ILP;
  double per_clk = units / (double)cmax;
  double total = units * nsm;
  double implied_mhz = (double)cmax / (ms * 1e3);
  printf("{\"op\": \"%s\", \"lanes_per_clk_per_sm\": %.2f, \"sass_instr_per_clk_per_sm\": %.2f, "
         "\"ops_per_s\": %.4e, \"ms\": %.4f, \"cycles\": %lld, \"implied_sm_mhz\": %.1f}\n",
         op_name[OP], per_clk, per_clk * op_instr[OP], total / (ms * 1e-3), ms, cmax, implied_mhz);
  delete[] hc; cudaFree(out); cudaFree(cyc);
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int nsm = p.multiProcessorCount;
  fprintf(stderr, "device %s, %d SMs\n", p.name, nsm);
  int rc = 0;
  rc |= run<IMAD_LO>(nsm, 2, 512);
  rc |= run<IMAD_HI>(nsm, 2, 512);
  rc |= run<IMAD_WIDE>(nsm, 2, 512);
  rc |= run<MADCHAIN>(nsm, 2, 512);
  rc |= run<IADD3_>(nsm, 2, 512);
  rc |= run<LOP3_>(nsm, 2, 512);
  rc |= run<VMIN_>(nsm, 2, 512);
  rc |= run<MIX_IMAD_IADD>(nsm, 2, 512);
  return rc;
}
