// Green's-function spectra on the device (S0 static part, S1 per frequency).
//
// eq:Hmn P:305 and P:308: H is three-level Toeplitz; its circulant embedding
// of size 2N_a per axis (reading R10) has first column K(h |o|), with
// K = K_s + K_d:
//   K_s(r) = 1/(4 pi r), K_s(0) = 0                         (eq:hgfs, eq:Hsmm P:321)
//   K_d(r) = (e^{-j k0 r} - 1)/(4 pi r), K_d(0) = -j k0/(4 pi)  (eq:hgfd, eq:Hdmm P:331)
// and 0 on the wrap slot o = N_a.  Because K is even along every axis, its
// 2N-point DFT is the (N+1)-point DCT-I of the octant samples,
//   H_hat[k] = sum_{i=0}^{N} c_i K[i] cos(pi i k / N),  c_0 = c_N = 1, c_i = 2,
// applied separably along z, x, y.  Each 1-D pass is a small dense
// contraction (a batched (N+1) x (N+1) GEMM on complex data with a real
// matrix), tiled in shared memory.  The static spectrum is built once in fp64;
// per frequency the dynamic part is sampled in fp64 (cancellation-free
// half-angle form, reading R11), rounded to the compute precision,
// transformed, added to H_hat_s and scaled by 1/M (the inverse-FFT
// normalisation is folded into the spectrum).  Octant layout: index
// ((ky (N_x+1) + kx) (N_z+1) + kz), z fastest.
#include <cmath>
#include <vector>

#include "aimx_internal.h"

namespace aimx {

namespace {

template <typename T> struct C2;
template <> struct C2<float> { using t = float2; };
template <> struct C2<double> { using t = double2; };

// sample[(j (Nx+1) + i)(Nz+1) + l] = K(h sqrt(i^2 + j^2 + l^2)), 0 on wrap slots
template <typename T, bool STATIC>
__global__ void k_sample(int Nx, int Ny, int Nz, double h, double k0,
                         typename C2<T>::t* __restrict__ out) {
  int64_t n = (int64_t)(Nx + 1) * (Ny + 1) * (Nz + 1);
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n) return;
  int l = (int)(idx % (Nz + 1));
  int64_t r2 = idx / (Nz + 1);
  int i = (int)(r2 % (Nx + 1));
  int j = (int)(r2 / (Nx + 1));
  double re = 0.0, im = 0.0;
  if (i < Nx && j < Ny && l < Nz) {
    int64_t q = (int64_t)i * i + (int64_t)j * j + (int64_t)l * l;
    const double inv4pi = 1.0 / (4.0 * kPi);
    if (STATIC) {
      if (q > 0) re = inv4pi / (h * sqrt((double)q));
    } else {
      if (q == 0) {
        im = -k0 * inv4pi;
      } else {
        double r = h * sqrt((double)q);
        double x = k0 * r;
        double s = sin(0.5 * x);
        re = -2.0 * s * s * inv4pi / r;
        im = -sin(x) * inv4pi / r;
      }
    }
  }
  typename C2<T>::t v;
  v.x = (T)re;
  v.y = (T)im;
  out[idx] = v;
}

// out[o][k][u] = sum_i C[k][i] in[o][i][u] (+ epilogue on the last pass:
// out = scale * (acc + add[idx])).  Tile 32 (k) x 64 (col = o*inner + u),
// chunks of 16 along i; 256 threads, 2 x 4 outputs each.
template <typename T>
__global__ void __launch_bounds__(256) k_dct_pass(int n1, int64_t outer, int64_t inner,
                                                  const T* __restrict__ C,
                                                  const typename C2<T>::t* __restrict__ in,
                                                  typename C2<T>::t* __restrict__ out,
                                                  const typename C2<T>::t* __restrict__ add,
                                                  T scale) {
  using T2 = typename C2<T>::t;
  __shared__ T sC[16][33];
  __shared__ T2 sI[16][65];
  const int tid = threadIdx.x;
  const int tk = tid >> 4;        // 0..15 -> k = k0 + tk*2 + {0,1}
  const int tc = tid & 15;        // 0..15 -> col = c0 + tc + 16*{0..3}
  const int64_t ncol = outer * inner;
  const int k0 = blockIdx.y * 32;
  const int64_t c0 = (int64_t)blockIdx.x * 64;
  T2 acc[2][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) { acc[a][b].x = 0; acc[a][b].y = 0; }
  for (int i0 = 0; i0 < n1; i0 += 16) {
    // C tile: 32 k x 16 i  (512 values, 2 per thread)
    for (int t = tid; t < 512; t += 256) {
      int kk = t >> 4, ii = t & 15;
      int k = k0 + kk, i = i0 + ii;
      sC[ii][kk] = (k < n1 && i < n1) ? C[(int64_t)k * n1 + i] : (T)0;
    }
    // In tile: 16 i x 64 col (1024 values, 4 per thread)
    for (int t = tid; t < 1024; t += 256) {
      int ii, cc;
      if (inner == 1) { ii = t & 15; cc = t >> 4; }   // contiguous along i
      else { cc = t & 63; ii = t >> 6; }             // contiguous along col
      int i = i0 + ii;
      int64_t col = c0 + cc;
      T2 v;
      v.x = 0; v.y = 0;
      if (i < n1 && col < ncol) {
        int64_t o = col / inner, u = col - o * inner;
        v = in[(o * n1 + i) * inner + u];
      }
      sI[ii][cc] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int ii = 0; ii < 16; ++ii) {
      T c_a = sC[ii][tk * 2], c_b = sC[ii][tk * 2 + 1];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        T2 v = sI[ii][tc + 16 * b];
        acc[0][b].x += c_a * v.x; acc[0][b].y += c_a * v.y;
        acc[1][b].x += c_b * v.x; acc[1][b].y += c_b * v.y;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    int k = k0 + tk * 2 + a;
    if (k >= n1) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int64_t col = c0 + tc + 16 * b;
      if (col >= ncol) continue;
      int64_t o = col / inner, u = col - o * inner;
      int64_t idx = (o * n1 + k) * inner + u;
      T2 r = acc[a][b];
      if (add) { r.x = scale * (r.x + add[idx].x); r.y = scale * (r.y + add[idx].y); }
      out[idx] = r;
    }
  }
}

template <typename T>
void dct_pass(int n1, int64_t outer, int64_t inner, const T* C, const void* in, void* out,
              const void* add, T scale, cudaStream_t s) {
  using T2 = typename C2<T>::t;
  int64_t ncol = outer * inner;
  dim3 grid((unsigned)((ncol + 63) / 64), (unsigned)((n1 + 31) / 32));
  k_dct_pass<T><<<grid, 256, 0, s>>>(n1, outer, inner, C, (const T2*)in, (T2*)out,
                                     (const T2*)add, scale);
  AIMX_CHECK_LAUNCH();
}

// 3-D DCT-I on the octant: z (contiguous), then x, then y.
template <typename T>
void dct3(SpectrumPlan& sp, const T* cx, const T* cy, const T* cz, void* a, void* b, void* out,
          const void* add, T scale, cudaStream_t s) {
  const int nx = sp.Nx + 1, ny = sp.Ny + 1, nz = sp.Nz + 1;
  dct_pass<T>(nz, (int64_t)ny * nx, 1, cz, a, b, nullptr, (T)1, s);
  dct_pass<T>(nx, ny, nz, cx, b, a, nullptr, (T)1, s);
  dct_pass<T>(ny, 1, (int64_t)nx * nz, cy, a, out, add, scale, s);
}

}  // namespace

void spectrum_plan_init(SpectrumPlan& sp, cudaStream_t s) {
  auto make = [&](int N, double*& d64, float*& d32) {
    int n1 = N + 1;
    std::vector<double> C((size_t)n1 * n1);
    std::vector<float> Cf((size_t)n1 * n1);
    for (int k = 0; k < n1; ++k)
      for (int i = 0; i < n1; ++i) {
        double ci = (i == 0 || i == N) ? 1.0 : 2.0;
        // cos(pi i k / N) with exact argument reduction modulo 2N
        int64_t m = ((int64_t)i * k) % (2 * N);
        double v = ci * std::cos(kPi * (double)m / (double)N);
        if (2 * m == N || 2 * m == 3 * N) v = 0.0;
        C[(size_t)k * n1 + i] = v;
        Cf[(size_t)k * n1 + i] = (float)v;
      }
    AIMX_CUDA(cudaMalloc(&d64, sizeof(double) * n1 * n1));
    AIMX_CUDA(cudaMalloc(&d32, sizeof(float) * n1 * n1));
    AIMX_CUDA(cudaMemcpyAsync(d64, C.data(), sizeof(double) * n1 * n1, cudaMemcpyHostToDevice, s));
    AIMX_CUDA(cudaMemcpyAsync(d32, Cf.data(), sizeof(float) * n1 * n1, cudaMemcpyHostToDevice, s));
    AIMX_CUDA(cudaStreamSynchronize(s));
  };
  make(sp.Nx, sp.cosx, sp.cosx_f);
  make(sp.Ny, sp.cosy, sp.cosy_f);
  make(sp.Nz, sp.cosz, sp.cosz_f);
  sp.noct = (int64_t)(sp.Nx + 1) * (sp.Ny + 1) * (sp.Nz + 1);
  AIMX_CUDA(cudaMalloc(&sp.work0, sizeof(double2) * sp.noct));
  AIMX_CUDA(cudaMalloc(&sp.work1, sizeof(double2) * sp.noct));
}

void spectrum_plan_free(SpectrumPlan& sp) {
  cudaFree(sp.cosx); cudaFree(sp.cosy); cudaFree(sp.cosz);
  cudaFree(sp.cosx_f); cudaFree(sp.cosy_f); cudaFree(sp.cosz_f);
  cudaFree(sp.work0); cudaFree(sp.work1);
  sp = SpectrumPlan{};
}

void spectrum_static(SpectrumPlan& sp, double2* out, cudaStream_t s) {
  int64_t n = sp.noct;
  k_sample<double, true><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sp.Nx, sp.Ny, sp.Nz, sp.h, 0.0,
                                                                   (double2*)sp.work0);
  AIMX_CHECK_LAUNCH();
  dct3<double>(sp, sp.cosx, sp.cosy, sp.cosz, sp.work0, sp.work1, out, nullptr, 1.0, s);
}

void spectrum_dynamic_f32(SpectrumPlan& sp, double k0, const float2* Hs, float scale, float2* out,
                          cudaStream_t s) {
  int64_t n = sp.noct;
  k_sample<float, false><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sp.Nx, sp.Ny, sp.Nz, sp.h, k0,
                                                                   (float2*)sp.work0);
  AIMX_CHECK_LAUNCH();
  dct3<float>(sp, sp.cosx_f, sp.cosy_f, sp.cosz_f, sp.work0, sp.work1, out, Hs, scale, s);
}

void spectrum_dynamic_f64(SpectrumPlan& sp, double k0, const double2* Hs, double scale,
                          double2* out, cudaStream_t s) {
  int64_t n = sp.noct;
  k_sample<double, false><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sp.Nx, sp.Ny, sp.Nz, sp.h, k0,
                                                                    (double2*)sp.work0);
  AIMX_CHECK_LAUNCH();
  dct3<double>(sp, sp.cosx, sp.cosy, sp.cosz, sp.work0, sp.work1, out, Hs, scale, s);
}

}  // namespace aimx
