// Green's-function spectra on the device (S0 static part, S1 per frequency).
//
// eq:Hmn P:305: H is three-level Toeplitz; its circulant embedding of
// size 2N_a per axis (reading R10) has first column K(h |o|), K = K_s + K_d
// (P:281):
//   K_s(r) = 1/(4 pi r), K_s(0) = 0                              (eq:hgfs, eq:Hsmm P:321)
//   K_d(r) = (e^{-j k0 r} - 1)/(4 pi r), K_d(0) = -j k0/(4 pi)    (eq:hgfd, eq:Hdmm P:331)
// and 0 on the wrap slot o = N_a.  K is even along every axis, so its 2N-point
// DFT is even as well and only the octant k in [0, N]^3 is kept.  Each axis is
// transformed by loading the N+1 octant samples of a line, rebuilding its even
// extension v[2N - i] = v[i] in shared memory and running the same Stockham
// FFT as the hot path (an exact DCT-I via FFT, O(N log N) per line, HBM-bound:
// one read + one write of the octant per axis).  The static spectrum is built
// once in fp64; per frequency the dynamic samples are computed in fp64 with the
// cancellation-free half-angle form (reading R11), rounded to the compute
// precision, transformed, added to H_hat_s and scaled by 1/M (the inverse-FFT
// normalisation is folded into the spectrum).  B frequencies per launch.
// Octant layout ((ky (N_z+1) + kz) (N_x+1) + kx), x fastest.
#include <cmath>
#include <vector>

#include "aimx_internal.h"
#include "fft.cuh"

namespace aimx {

namespace {

struct K0s { double v[kMaxBatch]; };

// sample[b][(j (Nz+1) + l)(Nx+1) + i] = K(h sqrt(i^2 + j^2 + l^2)), 0 on wrap slots
template <typename T, bool STATIC>
__global__ void k_sample(int Nx, int Ny, int Nz, int64_t noct, double h, K0s k0s,
                         typename CT<T>::T2* __restrict__ out) {
  using T2 = typename CT<T>::T2;
  const int b = blockIdx.y;
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= noct) return;
  const double k0 = k0s.v[b];
  int i = (int)(idx % (Nx + 1));
  int64_t r2 = idx / (Nx + 1);
  int l = (int)(r2 % (Nz + 1));
  int j = (int)(r2 / (Nz + 1));
  double re = 0.0, im = 0.0;
  if (i < Nx && j < Ny && l < Nz) {
    int64_t q = (int64_t)i * i + (int64_t)j * j + (int64_t)l * l;
    const double inv4pi = 1.0 / (4.0 * kPi);
    if (STATIC) {
      if (q > 0) re = inv4pi / (h * sqrt((double)q));
    } else if (q == 0) {
      im = -k0 * inv4pi;
    } else {
      double r = h * sqrt((double)q);
      double x = k0 * r;
      double s, c;
      sincos(0.5 * x, &s, &c);
      re = -2.0 * s * s * inv4pi / r;
      im = -2.0 * s * c * inv4pi / r;   // sin(x) = 2 sin(x/2) cos(x/2)
    }
  }
  out[(int64_t)b * noct + idx] = mk<T2>((T)re, (T)im);
}

// Row mode: lines contiguous (x axis), line l element i at l*n1 + i.
template <typename T, int L>
__global__ void __launch_bounds__(256) k_even_rows(int64_t nlines, int64_t noct,
                                                   const typename CT<T>::T2* __restrict__ in,
                                                   typename CT<T>::T2* __restrict__ out,
                                                   const typename CT<T>::T2* __restrict__ twg) {
  using T2 = typename CT<T>::T2;
  constexpr int N1 = L / 2 + 1;
  constexpr int R = (4096 / L) < 1 ? 1 : (4096 / L);
  constexpr int RS = L + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + R * RS;
  const int64_t l0 = (int64_t)blockIdx.x * R;
  const int nl = (int)min((int64_t)R, nlines - l0);
  const int64_t boff = (int64_t)blockIdx.y * noct;
  load_tw(tw, twg, L);
  const T2* __restrict__ src = in + boff + l0 * N1;
  for (int t = threadIdx.x; t < nl * N1; t += blockDim.x) {
    const int r = t / N1, i = t - r * N1;
    cp_async(b0 + r * RS + i, src + t);
  }
  cp_async_wait_all();
  __syncthreads();
  for (int t = threadIdx.x; t < nl * (L - N1); t += blockDim.x) {
    const int r = t / (L - N1), i = N1 + (t - r * (L - N1));
    b0[r * RS + i] = b0[r * RS + (L - i)];
  }
  __syncthreads();
  T2* s0 = b0;
  T2* s1 = b1;
  struct A { __device__ int operator()(int line, int idx) const { return line * RS + idx; } };
  smem_fft<T2, L, false>(s0, s1, nl, tw, A{});
  T2* __restrict__ dst = out + boff + l0 * N1;
  for (int t = threadIdx.x; t < nl * N1; t += blockDim.x) {
    const int r = t / N1, i = t - r * N1;
    dst[t] = s0[r * RS + i];
  }
}

// Column mode: element (o, i, u) at (o n1 + i) inner + u; tile of TW u's.
// Optional epilogue: out = scale * (v + add[idx]).
template <typename T, int L>
__global__ void __launch_bounds__(256) k_even_cols(int64_t inner, int TW, int64_t noct,
                                                   const typename CT<T>::T2* __restrict__ in,
                                                   typename CT<T>::T2* __restrict__ out,
                                                   const typename CT<T>::T2* __restrict__ twg,
                                                   const typename CT<T>::T2* __restrict__ add, T scale) {
  using T2 = typename CT<T>::T2;
  constexpr int N1 = L / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + L * TW;
  const int64_t u0 = (int64_t)blockIdx.x * TW;
  const int nu = (int)min((int64_t)TW, inner - u0);
  const int64_t o = blockIdx.y;
  const int64_t boff = (int64_t)blockIdx.z * noct;
  load_tw(tw, twg, L);
  const int64_t base = boff + o * N1 * inner + u0;
  for (int t = threadIdx.x; t < N1 * TW; t += blockDim.x) {
    const int i = t / TW, w = t - i * TW;
    if (w < nu) cp_async(b0 + t, in + base + (int64_t)i * inner + w);
    else b0[t] = mk<T2>(0, 0);
  }
  cp_async_wait_all();
  __syncthreads();
  for (int t = threadIdx.x; t < (L - N1) * TW; t += blockDim.x) {
    const int i = N1 + t / TW, w = t % TW;
    b0[i * TW + w] = b0[(L - i) * TW + w];
  }
  __syncthreads();
  T2* s0 = b0;
  T2* s1 = b1;
  smem_fft<T2, L, false>(s0, s1, TW, tw, ColAddr{TW});
  for (int t = threadIdx.x; t < N1 * TW; t += blockDim.x) {
    const int i = t / TW, w = t - i * TW;
    if (w >= nu) continue;
    const int64_t g = base + (int64_t)i * inner + w;
    T2 v = s0[t];
    if (add) {
      const T2 a = add[g - boff];
      v = mk<T2>(scale * (v.x + a.x), scale * (v.y + a.y));
    }
    out[g] = v;
  }
}

template <class K> void set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    AIMX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

template <typename T>
void even_rows(int L, int64_t nlines, int64_t noct, int B, const void* in, void* out, const void* tw,
               cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  AIMX_SWITCH_L(L, ({
    constexpr int R = (4096 / L) < 1 ? 1 : (4096 / L);
    size_t sm = sizeof(T2) * (L + 2 * R * (L + 1));
    set_smem(k_even_rows<T, L>, sm);
    dim3 g((unsigned)((nlines + R - 1) / R), (unsigned)B);
    k_even_rows<T, L><<<g, 256, sm, s>>>(nlines, noct, (const T2*)in, (T2*)out, (const T2*)tw);
  }));
  AIMX_CHECK_LAUNCH();
}

template <typename T>
void even_cols(int L, int64_t outer, int64_t inner, int64_t noct, int B, const void* in, void* out,
               const void* tw, const void* add, T scale, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  int TW = (int)(sizeof(T) == 4 ? 4096 : 2048) / L;
  TW = TW < 4 ? 4 : (TW > 256 ? 256 : TW);
  AIMX_SWITCH_L(L, ({
    size_t sm = sizeof(T2) * (L + 2 * (size_t)L * TW);
    set_smem(k_even_cols<T, L>, sm);
    dim3 g((unsigned)((inner + TW - 1) / TW), (unsigned)outer, (unsigned)B);
    k_even_cols<T, L><<<g, 256, sm, s>>>(inner, TW, noct, (const T2*)in, (T2*)out, (const T2*)tw,
                                         (const T2*)add, scale);
  }));
  AIMX_CHECK_LAUNCH();
}

// 3-D even-extension transform on the octant [B][y][z][x]: x rows, z cols, y cols.
template <typename T>
void dct3(SpectrumPlan& sp, int B, void** tw, void* a, void* b, void* out, const void* add, T scale,
          cudaStream_t s) {
  const int64_t nx = sp.Nx + 1, ny = sp.Ny + 1, nz = sp.Nz + 1, no = sp.noct;
  even_rows<T>(2 * sp.Nx, ny * nz, no, B, a, b, tw[0], s);
  even_cols<T>(2 * sp.Nz, ny, nx, no, B, b, a, tw[2], nullptr, (T)1, s);
  even_cols<T>(2 * sp.Ny, 1, nz * nx, no, B, a, out, tw[1], add, scale, s);
}

}  // namespace

void spectrum_plan_init(SpectrumPlan& sp, int batch, cudaStream_t s) {
  auto make = [&](int L, int a) {
    std::vector<double2> d(L);
    std::vector<float2> f(L);
    for (int m = 0; m < L; ++m) {
      double ang = 2.0 * kPi * (double)m / (double)L;
      double re = std::cos(ang), im = -std::sin(ang);
      if (4 * m == L || 4 * m == 3 * L) re = 0.0;
      if (2 * m == L || m == 0) im = 0.0;
      d[m] = make_double2(re, im);
      f[m] = make_float2((float)re, (float)im);
    }
    AIMX_CUDA(cudaMalloc(&sp.tw64[a], sizeof(double2) * L));
    AIMX_CUDA(cudaMalloc(&sp.tw32[a], sizeof(float2) * L));
    AIMX_CUDA(cudaMemcpyAsync(sp.tw64[a], d.data(), sizeof(double2) * L, cudaMemcpyHostToDevice, s));
    AIMX_CUDA(cudaMemcpyAsync(sp.tw32[a], f.data(), sizeof(float2) * L, cudaMemcpyHostToDevice, s));
    AIMX_CUDA(cudaStreamSynchronize(s));
  };
  make(2 * sp.Nx, 0);
  make(2 * sp.Ny, 1);
  make(2 * sp.Nz, 2);
  sp.noct = (int64_t)(sp.Nx + 1) * (sp.Ny + 1) * (sp.Nz + 1);
  sp.batch = batch < 1 ? 1 : batch;
  AIMX_CUDA(cudaMalloc(&sp.work0, sizeof(double2) * sp.noct * sp.batch));
  AIMX_CUDA(cudaMalloc(&sp.work1, sizeof(double2) * sp.noct * sp.batch));
}

void spectrum_plan_free(SpectrumPlan& sp) {
  for (int a = 0; a < 3; ++a) {
    cudaFree(sp.tw64[a]);
    cudaFree(sp.tw32[a]);
  }
  cudaFree(sp.work0);
  cudaFree(sp.work1);
  sp = SpectrumPlan{};
}

void spectrum_static(SpectrumPlan& sp, double2* out, cudaStream_t s) {
  K0s k{};
  k_sample<double, true><<<dim3((unsigned)((sp.noct + 255) / 256), 1), 256, 0, s>>>(
      sp.Nx, sp.Ny, sp.Nz, sp.noct, sp.h, k, (double2*)sp.work0);
  AIMX_CHECK_LAUNCH();
  dct3<double>(sp, 1, sp.tw64, sp.work0, sp.work1, out, nullptr, 1.0, s);
}

void spectrum_dynamic_f32(SpectrumPlan& sp, int B, const double* k0, const float2* Hs, float scale,
                          float2* out, cudaStream_t s) {
  if (B > sp.batch || B > kMaxBatch) throw Error(AIMX_E_INTERNAL, "spectrum batch too large");
  K0s k{};
  for (int b = 0; b < B; ++b) k.v[b] = k0[b];
  k_sample<float, false><<<dim3((unsigned)((sp.noct + 255) / 256), (unsigned)B), 256, 0, s>>>(
      sp.Nx, sp.Ny, sp.Nz, sp.noct, sp.h, k, (float2*)sp.work0);
  AIMX_CHECK_LAUNCH();
  dct3<float>(sp, B, sp.tw32, sp.work0, sp.work1, out, Hs, scale, s);
}

void spectrum_dynamic_f64(SpectrumPlan& sp, int B, const double* k0, const double2* Hs,
                          double scale, double2* out, cudaStream_t s) {
  if (B > sp.batch || B > kMaxBatch) throw Error(AIMX_E_INTERNAL, "spectrum batch too large");
  K0s k{};
  for (int b = 0; b < B; ++b) k.v[b] = k0[b];
  k_sample<double, false><<<dim3((unsigned)((sp.noct + 255) / 256), (unsigned)B), 256, 0, s>>>(
      sp.Nx, sp.Ny, sp.Nz, sp.noct, sp.h, k, (double2*)sp.work0);
  AIMX_CHECK_LAUNCH();
  dct3<double>(sp, B, sp.tw64, sp.work0, sp.work1, out, Hs, scale, s);
}

}  // namespace aimx
