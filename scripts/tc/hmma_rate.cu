// Legacy tensor-core (mma.sync / HMMA) issue rate on sm_100a: tf32 m16n8k8 and
// bf16 m16n8k16, ILP independent accumulators per warp, grid = 148 x CTAs/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma_rate hmma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int ILP, bool BF16>
__global__ void k_rate(float* out, int iters) {
  float d[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.f;
  uint32_t a0 = threadIdx.x, a1 = a0 ^ 5, a2 = a0 ^ 9, a3 = a0 ^ 3, b0 = a0 * 7, b1 = a0 * 3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if constexpr (BF16)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <int ILP, bool BF16>
void run(int ctas_per_sm, int threads) {
  float* out;
  cudaMalloc(&out, 4096);
  const int iters = 4096, grid = 148 * ctas_per_sm;
  k_rate<ILP, BF16><<<grid, threads>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<ILP, BF16><<<grid, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop_per_mma = BF16 ? 2.0 * 16 * 8 * 16 : 2.0 * 16 * 8 * 8;
  const double mmas = (double)grid * (threads / 32) * iters * ILP;
  printf("%s ILP=%d ctas/SM=%d threads=%d: %.3f ms, %.1f TFLOP/s, %.2f mma/clk/SM at 1.92 GHz\n",
         BF16 ? "bf16 m16n8k16" : "tf32 m16n8k8 ", ILP, ctas_per_sm, threads, ms,
         mmas * flop_per_mma / ms / 1e9, mmas / (ms * 1e-3) / 148 / 1.92e9);
  cudaFree(out);
}

int main() {
  run<8, false>(4, 128);
  run<8, false>(8, 128);
  run<4, false>(8, 128);
  run<16, false>(4, 128);
  run<8, true>(4, 128);
  run<8, true>(8, 128);
  return 0;
}
