// pipe_mix.cu — which pipes run concurrently on sm_100a (B200)?
//
// Sustained throughput (lanes per SM clock) of: DFMA alone, IMAD.WIDE alone,
// DFMA + IMAD.WIDE interleaved, IADD3 alone (chained, not foldable),
// VIADDMNMX alone, IMAD.WIDE + IADD3 + DFMA.  Decides whether the idle
// FP64 pipe could take part of the classical product's partial products
// ("Roofline denominators").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix pipe_mix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ILP = 8;
constexpr int ITERS = 2048;
enum { DFMA_, IWIDE_, DFMA_IWIDE, IADD3_, VMNMX_, IWIDE_IADD3_DFMA, IWIDE2_DFMA1, NOPS };
static const char* nm[NOPS] = {"dfma", "imad_wide", "dfma+imad_wide", "iadd3_chain", "viaddmnmx_chain",
                               "imad_wide+iadd3+dfma", "2imad_wide+dfma"};

template <int OP>
__global__ void kern(uint32_t* out, uint32_t seed, long long* cyc) {
  uint32_t r[ILP], s[ILP];
  double d[ILP];
#pragma unroll
  for (int k = 0; k < ILP; k++) {
    r[k] = seed + threadIdx.x * 7 + k;
    s[k] = seed ^ (k * 0x9e3779b9u);
    d[k] = 1.0 + k * 1e-3 + threadIdx.x * 1e-6;
  }
  const uint32_t a = seed * 3 + 1;
  const double x = 1.0000001, y = 1e-9;
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int k = 0; k < ILP; k++) {
      if (OP == DFMA_ || OP == DFMA_IWIDE || OP == IWIDE_IADD3_DFMA || OP == IWIDE2_DFMA1)
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[k]) : "d"(x), "d"(y));
      if (OP == IWIDE_ || OP == DFMA_IWIDE || OP == IWIDE_IADD3_DFMA || OP == IWIDE2_DFMA1) {
        uint64_t w;
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(r[k]), "r"(a), "l"(((uint64_t)s[k] << 32) | r[k]));
        r[k] = (uint32_t)w; s[k] = (uint32_t)(w >> 32);
      }
      if (OP == IWIDE2_DFMA1) {
        uint64_t w;
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(s[k]), "r"(a), "l"(((uint64_t)r[k] << 32) | s[k]));
        r[k] = (uint32_t)w; s[k] = (uint32_t)(w >> 32);
      }
      if (OP == IADD3_ || OP == IWIDE_IADD3_DFMA)
        asm volatile("add.u32 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
      if (OP == IADD3_) asm volatile("add.u32 %0, %0, %1;" : "+r"(s[k]) : "r"(r[k]));
      if (OP == VMNMX_) {
        asm volatile("{ .reg .u32 t; add.u32 t, %0, %1; min.u32 %0, t, %0; }" : "+r"(r[k]) : "r"(a));
      }
    }
  }
  long long c1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < ILP; k++) acc ^= r[k] ^ s[k] ^ (uint32_t)__double2loint(d[k]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

template <int OP>
void run(int nsm) {
  const int ctas = 2, threads = 512, grid = nsm * ctas;
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, sizeof(uint32_t) * grid * threads);
  cudaMalloc(&cyc, sizeof(long long) * grid);
  kern<OP><<<grid, threads>>>(out, 1, cyc);
  cudaDeviceSynchronize();
  kern<OP><<<grid, threads>>>(out, 2, cyc);
  cudaDeviceSynchronize();
  long long h[4096];
  cudaMemcpy(h, cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  long long cmax = 0;
  for (int i = 0; i < grid; i++) cmax = h[i] > cmax ? h[i] : cmax;
  const double units = (double)ctas * threads * ITERS * ILP;
  printf("{\"op\": \"%s\", \"iterations_per_clk_per_sm\": %.2f, \"cycles\": %lld}\n", nm[OP], units / cmax, cmax);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  fprintf(stderr, "device %s, %d SMs\n", p.name, p.multiProcessorCount);
  run<DFMA_>(p.multiProcessorCount);
  run<IWIDE_>(p.multiProcessorCount);
  run<DFMA_IWIDE>(p.multiProcessorCount);
  run<IADD3_>(p.multiProcessorCount);
  run<VMNMX_>(p.multiProcessorCount);
  run<IWIDE_IADD3_DFMA>(p.multiProcessorCount);
  run<IWIDE2_DFMA1>(p.multiProcessorCount);
  return 0;
}
