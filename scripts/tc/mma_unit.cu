// Standalone unit test of one tcgen05.mma kind::tf32 (M=64, N=16, K=8) with
// A (64 x 8) MN-major 128B-swizzled and B (8 x 16) MN-major unswizzled in
// shared memory; D read back with tcgen05.ld 32x32b.x16.  Variants of the
// descriptor fields come from the command line to pin the encoding.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mkdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | ((uint64_t)layout << 61);
}

struct Args { uint32_t a_lbo, a_sbo, a_layout, b_lbo, b_sbo, b_layout, idesc; int a_mode, b_mode; };

__global__ void k(const float* A, const float* B, float* D, Args g) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024u - (su32(sm) & 1023u)) & 1023u);
  float* sA = (float*)base;            // 2 KB
  float* sB = (float*)(base + 2048);   // 512 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  // A[m][k] m<64 k<8
  for (int i = tid; i < 64 * 8; i += 128) {
    const int m = i / 8, kk = i % 8;
    int off;   // float index
    if (g.a_mode == 0) {   // SW128 MN-major: atom m/32 at 1024 B, row kk at 128 B, chunk ((m%32)/4 ^ kk) at 16 B
      off = ((m / 32) * 1024 + kk * 128 + ((((m % 32) / 4) ^ kk) << 4)) / 4 + (m % 4);
    } else if (g.a_mode == 2) {   // no swizzle K-major: core (8 m x 4 k): (m%8)*16 + (m/8)*128 + (k/4)*1024 + (k%4)*4
      off = ((m % 8) * 16 + (m / 8) * 128 + (kk / 4) * 1024) / 4 + (kk % 4);
    } else {               // no swizzle MN-major: core (8 k x 4 m): (m/4) * 128 + kk * 16 + (m%4) * 4
      off = ((m / 4) * 128 + kk * 16) / 4 + (m % 4);
    }
    sA[off] = A[m * 8 + kk];
  }
  for (int i = tid; i < 8 * 16; i += 128) {
    const int kk = i / 16, n = i % 16;
    int off;
    if (g.b_mode == 0) off = ((n / 4) * 128 + kk * 16) / 4 + (n % 4);   // no swizzle MN-major
    else off = ((n % 8) * 16 + (n / 8) * 128 + (kk / 4) * 256) / 4 + (kk % 4);  // K-major core (8 n x 4 k): n-blocks 128 B, k-blocks 256 B
    sB[off] = B[kk * 16 + n];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  if (g.a_mode == 9) {   // tcgen05.st / ld roundtrip: value = 1000 * lane + col
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint((float)(1000 * (32 * w + lane) + j));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                 ::"r"(tmem + ((uint32_t)(32 * w) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                 "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0 && g.a_mode != 9) {
    const uint64_t ad = mkdesc(su32(sA), g.a_lbo, g.a_sbo, g.a_layout);
    const uint64_t bd = mkdesc(su32(sB), g.b_lbo, g.b_sbo, g.b_layout);
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                 "l"(ad), "l"(bd), "r"(g.idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)) : "memory");
  }
  if (g.a_mode != 9) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                 "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(tmem + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  // raw dump: D[warp][lane][16]
  for (int j = 0; j < 16; ++j) D[(w * 32 + lane) * 16 + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tmem));
}

int main(int argc, char** argv) {
  float hA[64 * 8], hB[8 * 16], ref[64 * 16];
  for (int m = 0; m < 64; ++m) for (int kk = 0; kk < 8; ++kk) hA[m * 8 + kk] = (float)((m * 3 + kk * 7) % 11 - 5);
  for (int kk = 0; kk < 8; ++kk) for (int n = 0; n < 16; ++n) hB[kk * 16 + n] = (float)((kk * 5 + n * 3) % 7 - 3);
  for (int m = 0; m < 64; ++m) for (int n = 0; n < 16; ++n) { double s = 0; for (int kk = 0; kk < 8; ++kk) s += hA[m * 8 + kk] * hB[kk * 16 + n]; ref[m * 16 + n] = (float)s; }
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, 128 * 16 * 4);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  const uint32_t base_idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((64u >> 4) << 24);
  struct V { const char* name; Args a; } vs[] = {
    {"A sw128 MN lbo1024 sbo2048 | B none MN lbo512 sbo128", {1024, 2048, 2, 512, 128, 0, base_idesc | (1u << 15) | (1u << 16), 0, 0}},
    {"A sw128 MN lbo2048 sbo1024 | B none MN lbo512 sbo128", {2048, 1024, 2, 512, 128, 0, base_idesc | (1u << 15) | (1u << 16), 0, 0}},
    {"A sw128 MN lbo1024 sbo2048 | B none MN lbo128 sbo512", {1024, 2048, 2, 128, 512, 0, base_idesc | (1u << 15) | (1u << 16), 0, 0}},
    {"A sw128 MN lbo2048 sbo1024 | B none MN lbo128 sbo512", {2048, 1024, 2, 128, 512, 0, base_idesc | (1u << 15) | (1u << 16), 0, 0}},
    {"A none MN lbo2048 sbo128 | B none MN lbo512 sbo128", {2048, 128, 0, 512, 128, 0, base_idesc | (1u << 15) | (1u << 16), 1, 0}},
    {"A none MN lbo128 sbo2048 | B none MN lbo128 sbo512", {128, 2048, 0, 128, 512, 0, base_idesc | (1u << 15) | (1u << 16), 1, 0}},
    {"K/K none: A lbo1024 sbo128 | B lbo256 sbo128", {1024, 128, 0, 256, 128, 0, base_idesc, 2, 1}},
    {"K/K none: A lbo128 sbo1024 | B lbo128 sbo256", {128, 1024, 0, 128, 256, 0, base_idesc, 2, 1}},
    {"tcgen05.st/ld roundtrip", {0, 0, 0, 0, 0, 0, 0, 9, 0}},
  };
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  for (auto& v : vs) {
    cudaMemset(D, 0, 128 * 16 * 4);
    k<<<1, 128, 8192>>>(A, B, D, v.a);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: CUDA error %s\n", v.name, cudaGetErrorString(e)); return 1; }
    float hD[128 * 16];
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    // expected: row m in lane (m % 16) + 32 (m / 16)
    double err = 0, mx = 0; int bad = 0;
    for (int m = 0; m < 64; ++m) for (int n = 0; n < 16; ++n) {
      const float got = hD[((m % 16) + 32 * (m / 16)) * 16 + n];
      err = fmax(err, fabs(got - ref[m * 16 + n])); mx = fmax(mx, fabs(ref[m * 16 + n]));
      if (got != ref[m * 16 + n]) ++bad;
    }
    printf("%-60s max|err| %.3g (max|ref| %.3g), %d of 1024 wrong\n", v.name, err, mx, bad);
    int nz = 0;
    for (int l = 0; l < 128; ++l) for (int j = 0; j < 16; ++j) if (hD[l * 16 + j] != 0.f) { if (nz < 12) printf("   nz lane %d col %d = %g\n", l, j, hD[l * 16 + j]); ++nz; }
    printf("   nonzero entries in the dump: %d\n", nz);
    if (v.a.a_mode == 9) { int ok = 1; for (int l = 0; l < 128; ++l) for (int j = 0; j < 16; ++j) ok &= hD[l * 16 + j] == (float)(1000 * l + j); printf("   roundtrip %s\n", ok ? "OK" : "WRONG"); }
    if (bad) {
      printf("  row0 got:"); for (int n = 0; n < 16; ++n) printf(" %g", hD[n]); printf("\n  row0 ref:"); for (int n = 0; n < 16; ++n) printf(" %g", ref[n]); printf("\n");
      printf("  row1 got:"); for (int n = 0; n < 16; ++n) printf(" %g", hD[16 + n]); printf("\n  row1 ref:"); for (int n = 0; n < 16; ++n) printf(" %g", ref[16 + n]); printf("\n");
    }
  }
  return 0;
}
