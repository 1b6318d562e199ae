// Batched GMRES building blocks (P:727-728 GMRES with a
// relative residual of 1e-4; P:340-359 diagonal preconditioner from the static
// self terms).  B frequency points iterate together: column b of every [B][N]
// block belongs to frequency b.  Reductions are fixed-order (one CTA per
// (vector, column)), so results are deterministic; dot products accumulate in
// fp64 in both precisions.
#include "aimx_internal.h"
#include "fft.cuh"

namespace aimx {

namespace {

template <typename T2> __device__ __forceinline__ double2 to_d(const T2& v) { return make_double2(v.x, v.y); }

// out[b][n] (+)= in[b][n] / M_b[n],  M_b[n] = j alpha_b (dA[n] - beta_b dR[n])
template <typename T2>
__global__ void k_pc(int B, int64_t N, const T2* __restrict__ in, T2* __restrict__ out, const double* __restrict__ dA,
                     const double* __restrict__ dR, PcArgs pa, int accumulate) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * N) return;
  const int b = (int)(i / N);
  const int64_t n = i - (int64_t)b * N;
  const double m = pa.alpha_im[b] * (dA[n] - pa.beta[b] * dR[n]);   // M = j m
  const double2 v = to_d(in[i]);
  double2 r = make_double2(v.y / m, -v.x / m);                      // v / (j m) = -j v / m
  if (accumulate) {
    const double2 o = to_d(out[i]);
    r.x += o.x;
    r.y += o.y;
  }
  out[i] = mk<T2>(r.x, r.y);
}

// out[v][b] = sum_n conj(V[v][b][n]) W[b][n], v < nv (V vectors nv apart by vstride)
template <typename T2>
__global__ void __launch_bounds__(256) k_dots(int64_t N, const T2* __restrict__ V, int64_t vstride,
                                              const T2* __restrict__ W, double2* __restrict__ out, int B) {
  pdl_wait();
  pdl_trigger();
  const int v = blockIdx.x, b = blockIdx.y;
  const T2* a = V + v * vstride + (int64_t)b * N;
  const T2* w = W + (int64_t)b * N;
  double sx = 0.0, sy = 0.0;
  for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
    const double2 p = to_d(a[n]), q = to_d(w[n]);
    sx += p.x * q.x + p.y * q.y;
    sy += p.x * q.y - p.y * q.x;
  }
  __shared__ double rx[256], ry[256];
  rx[threadIdx.x] = sx;
  ry[threadIdx.x] = sy;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      rx[threadIdx.x] += rx[threadIdx.x + o];
      ry[threadIdx.x] += ry[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[(int64_t)v * B + b] = make_double2(rx[0], ry[0]);
}

// W[b][n] = (mode ? 0 : W[b][n]) - sign * sum_v coef[v][b] V[v][b][n]   (mode 1: sign = -1 -> plain sum)
template <typename T2>
__global__ void k_lincomb(int nv, int B, int64_t N, const T2* __restrict__ V, int64_t vstride,
                          const double2* __restrict__ coef, T2* __restrict__ W, int mode) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * N) return;
  const int b = (int)(i / N);
  double2 acc = mode ? make_double2(0.0, 0.0) : to_d(W[i]);
  const double sg = mode ? 1.0 : -1.0;
  for (int v = 0; v < nv; ++v) {
    const double2 c = coef[(int64_t)v * B + b], p = to_d(V[v * vstride + i]);
    acc.x += sg * (c.x * p.x - c.y * p.y);
    acc.y += sg * (c.x * p.y + c.y * p.x);
  }
  W[i] = mk<T2>(acc.x, acc.y);
}

// out[b][n] = s[b] * W[b][n]
template <typename T2>
__global__ void k_colscale(int B, int64_t N, const T2* __restrict__ W, const double* __restrict__ s, T2* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * N) return;
  const double f = s[i / N];
  const double2 w = to_d(W[i]);
  out[i] = mk<T2>(f * w.x, f * w.y);
}

// out_b = W_b / sqrt(n_b.x) (0 where n_b.x = 0): the Arnoldi normalisation
// with the norm left on the device
template <typename T2>
__global__ void k_colscale_rsqrt(int B, int64_t N, const T2* __restrict__ W, const double2* __restrict__ n2,
                                 T2* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * N) return;
  const double q = n2[i / N].x;
  const double f = q > 0.0 ? 1.0 / sqrt(q) : 0.0;
  const double2 w = to_d(W[i]);
  out[i] = mk<T2>(f * w.x, f * w.y);
}

// y += a t (a real)
template <typename T2>
__global__ void k_axpy(int64_t n, double a, const T2* __restrict__ t, T2* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 u = to_d(t[i]), v = to_d(y[i]);
  y[i] = mk<T2>(v.x + a * u.x, v.y + a * u.y);
}

// y += a t (a complex)
template <typename T2>
__global__ void k_caxpy(int64_t n, double ar, double ai, const T2* __restrict__ t, T2* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 u = to_d(t[i]), v = to_d(y[i]);
  y[i] = mk<T2>(v.x + ar * u.x - ai * u.y, v.y + ar * u.y + ai * u.x);
}

// out = a - b
template <typename T2>
__global__ void k_sub(int64_t n, const T2* __restrict__ a, const T2* __restrict__ b, T2* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = mk<T2>(a[i].x - b[i].x, a[i].y - b[i].y);
}

// d[m] = src[diag[m]]
__global__ void k_take(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ src, double* __restrict__ d) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) d[i] = src[idx[i]];
}

unsigned nb256(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

void gm_pc(bool f32, int B, int64_t N, const void* in, void* out, const double* dA, const double* dR, const PcArgs& pa,
           bool accumulate, cudaStream_t s) {
  if (f32) launch_pdl(k_pc<float2>, dim3(nb256(B * N)), dim3(256), 0, s, B, N, (const float2*)in, (float2*)out, dA, dR, pa, accumulate);
  else launch_pdl(k_pc<double2>, dim3(nb256(B * N)), dim3(256), 0, s, B, N, (const double2*)in, (double2*)out, dA, dR, pa, accumulate);
  AIMX_CHECK_LAUNCH();
}
void gm_dots(bool f32, int nv, int B, int64_t N, const void* V, int64_t vstride, const void* W, double2* out,
             cudaStream_t s) {
  if (nv <= 0) return;
  dim3 g((unsigned)nv, (unsigned)B);
  if (f32) launch_pdl(k_dots<float2>, dim3(g), dim3(256), 0, s, N, (const float2*)V, vstride, (const float2*)W, out, B);
  else launch_pdl(k_dots<double2>, dim3(g), dim3(256), 0, s, N, (const double2*)V, vstride, (const double2*)W, out, B);
  AIMX_CHECK_LAUNCH();
}
void gm_lincomb(bool f32, int nv, int B, int64_t N, const void* V, int64_t vstride, const double2* coef, void* W,
                bool assign, cudaStream_t s) {
  if (f32)
    launch_pdl(k_lincomb<float2>, dim3(nb256(B * N)), dim3(256), 0, s, nv, B, N, (const float2*)V, vstride, coef, (float2*)W, assign);
  else
    launch_pdl(k_lincomb<double2>, dim3(nb256(B * N)), dim3(256), 0, s, nv, B, N, (const double2*)V, vstride, coef, (double2*)W, assign);
  AIMX_CHECK_LAUNCH();
}
void gm_colscale(bool f32, int B, int64_t N, const void* W, const double* sc, void* out, cudaStream_t s) {
  if (f32) launch_pdl(k_colscale<float2>, dim3(nb256(B * N)), dim3(256), 0, s, B, N, (const float2*)W, sc, (float2*)out);
  else launch_pdl(k_colscale<double2>, dim3(nb256(B * N)), dim3(256), 0, s, B, N, (const double2*)W, sc, (double2*)out);
  AIMX_CHECK_LAUNCH();
}
void gm_colscale_rsqrt(bool f32, int B, int64_t N, const void* W, const double2* n2, void* out, cudaStream_t s) {
  if (f32) launch_pdl(k_colscale_rsqrt<float2>, dim3(nb256(B * N)), dim3(256), 0, s, B, N, (const float2*)W, n2, (float2*)out);
  else launch_pdl(k_colscale_rsqrt<double2>, dim3(nb256(B * N)), dim3(256), 0, s, B, N, (const double2*)W, n2, (double2*)out);
  AIMX_CHECK_LAUNCH();
}
void gm_axpy(bool f32, int64_t n, double a, const void* t, void* y, cudaStream_t s) {
  if (f32) launch_pdl(k_axpy<float2>, dim3(nb256(n)), dim3(256), 0, s, n, a, (const float2*)t, (float2*)y);
  else launch_pdl(k_axpy<double2>, dim3(nb256(n)), dim3(256), 0, s, n, a, (const double2*)t, (double2*)y);
  AIMX_CHECK_LAUNCH();
}
void gm_caxpy(bool f32, int64_t n, double ar, double ai, const void* t, void* y, cudaStream_t s) {
  if (f32) launch_pdl(k_caxpy<float2>, dim3(nb256(n)), dim3(256), 0, s, n, ar, ai, (const float2*)t, (float2*)y);
  else launch_pdl(k_caxpy<double2>, dim3(nb256(n)), dim3(256), 0, s, n, ar, ai, (const double2*)t, (double2*)y);
  AIMX_CHECK_LAUNCH();
}
void gm_sub(bool f32, int64_t n, const void* a, const void* b, void* out, cudaStream_t s) {
  if (f32) launch_pdl(k_sub<float2>, dim3(nb256(n)), dim3(256), 0, s, n, (const float2*)a, (const float2*)b, (float2*)out);
  else launch_pdl(k_sub<double2>, dim3(nb256(n)), dim3(256), 0, s, n, (const double2*)a, (const double2*)b, (double2*)out);
  AIMX_CHECK_LAUNCH();
}
void gm_take(int64_t n, const int64_t* idx, const double* src, double* d, cudaStream_t s) {
  launch_pdl(k_take, dim3(nb256(n)), dim3(256), 0, s, n, idx, src, d);
  AIMX_CHECK_LAUNCH();
}

}  // namespace aimx
