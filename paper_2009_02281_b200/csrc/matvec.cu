// The AIMx hot path on the B200 (S2-S5), batched over B frequency points:
//
//   k_gather      S2: projection P x as a gather over the transposed
//                 (node-major) stencil CSR -- a group of G lanes per occupied
//                 grid node, fixed-order shuffle reduction, no atomics -- into
//                 dense occupied x-lines S[line][x][4]
//   k_xfwd        zero-padded forward FFT along x of the occupied lines
//   k_yfwd        forward FFT along y (input rows y < N_y, zero padded)
//   k_zconv       forward FFT along z, times the spectrum H_hat (octant,
//                 already scaled by 1/M), inverse FFT along z, cropped to z < N_z
//   k_yinv        inverse FFT along y, cropped to y < N_y (occupied lines only)
//   k_xinv        inverse FFT along x, cropped to x < N_x -> potentials phi
//   k_interp_near S4 + S5: warp per RWG (testing function): interpolation
//                 W = P^T of the 4 potentials on its (n+1)^3 stencil, plus the
//                 near-region row of C = L_s,NR - L_s,P (read once for all B
//                 right-hand sides), plus the EFIE combine
//                 y = -j w mu0 (y^A - k0^-2 y^rho).
//
// P:198-200 (W H P, "accelerated with FFTs", applied on the entire grid);
// eq:LAIMx P:283; eq:EFIEAIMx P:288.  Grid data are complex, 4 channels
// (x, y, z, rho) innermost: element ((z * Ny' + y) * Nx' + x) * 4 + c.
// Pruning (exact, reading R12): lines/planes with no occupied node are never
// transformed; their data are identically zero and are never read as input.
#include <algorithm>

#include "aimx_internal.h"
#include "fft.cuh"

namespace aimx {

namespace {

template <typename T> constexpr int rows_x(int L) {
  int r = (sizeof(T) == 4 ? 4096 : 2048) / (4 * L);
  return r < 1 ? 1 : (r > 32 ? 32 : r);
}

// ------------------------------------------------------------------ S2 gather
template <typename T, int G>
__global__ void __launch_bounds__(256) k_gather(HotDev h, const typename CT<T>::T2* __restrict__ x,
                                                int64_t xstride) {
  using T2 = typename CT<T>::T2;
  using T4 = typename CT<T>::T4;
  const int b = blockIdx.y;
  const int gl = threadIdx.x & (G - 1);
  const int q = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G);
  const bool act = q < h.nocc;
  const T2* __restrict__ xb = x + b * xstride;
  T2 a0 = mk<T2>(0, 0), a1 = a0, a2 = a0, a3 = a0;
  if (act) {
    const T4* __restrict__ ew = (const T4*)h.ent_w;
    const int e1 = h.node_ptr[q + 1];
#pragma unroll 4
    for (int e = h.node_ptr[q] + gl; e < e1; e += G) {
      const T4 w = ew[e];
      const T2 xv = xb[h.ent_rwg[e]];
      a0.x += w.x * xv.x; a0.y += w.x * xv.y;
      a1.x += w.y * xv.x; a1.y += w.y * xv.y;
      a2.x += w.z * xv.x; a2.y += w.z * xv.y;
      a3.x += w.w * xv.x; a3.y += w.w * xv.y;
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    a0.x += __shfl_xor_sync(0xffffffffu, a0.x, o); a0.y += __shfl_xor_sync(0xffffffffu, a0.y, o);
    a1.x += __shfl_xor_sync(0xffffffffu, a1.x, o); a1.y += __shfl_xor_sync(0xffffffffu, a1.y, o);
    a2.x += __shfl_xor_sync(0xffffffffu, a2.x, o); a2.y += __shfl_xor_sync(0xffffffffu, a2.y, o);
    a3.x += __shfl_xor_sync(0xffffffffu, a3.x, o); a3.y += __shfl_xor_sync(0xffffffffu, a3.y, o);
  }
  if (act && gl == 0) {
    T2* dst = (T2*)h.S + b * h.sS + ((int64_t)h.node_line[q] * h.Nx + h.node_lin[q] % h.Nx) * 4;
    dst[0] = a0; dst[1] = a1; dst[2] = a2; dst[3] = a3;
  }
}

// ------------------------------------------------------------------ x-fwd
template <typename T, int L>
__global__ void __launch_bounds__(256) k_xfwd(HotDev h) {
  using T2 = typename CT<T>::T2;
  constexpr int ROWS = rows_x<T>(L);
  constexpr int RS = (L + 1) * 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + ROWS * RS;
  const int b = blockIdx.y;
  const int l0 = blockIdx.x * ROWS;
  const int nrows = min(ROWS, h.nlines - l0);
  const int Nx = h.Nx;
  load_tw(tw, (const T2*)h.twx, L);
  const T2* __restrict__ in = (const T2*)h.S + b * h.sS + (int64_t)l0 * Nx * 4;
  for (int i = threadIdx.x; i < nrows * Nx * 4; i += blockDim.x) {
    const int r = i / (Nx * 4), e = i - r * (Nx * 4);
    cp_async(b0 + r * RS + e, in + i);
  }
  for (int i = threadIdx.x; i < nrows * (L - Nx) * 4; i += blockDim.x) {
    const int r = i / ((L - Nx) * 4), e = Nx * 4 + i - r * ((L - Nx) * 4);
    b0[r * RS + e] = mk<T2>(0, 0);
  }
  cp_async_wait_all();
  __syncthreads();
  T2* src = b0;
  T2* dst = b1;
  smem_fft<T2, L, false>(src, dst, nrows * 4, tw, RowAddr<L>{});
  T2* __restrict__ out = (T2*)h.bufA + b * h.sA;
  for (int r = 0; r < nrows; ++r) {
    const int64_t base = (int64_t)h.line_id[l0 + r] * L * 4;
    for (int i = threadIdx.x; i < L * 4; i += blockDim.x) out[base + i] = src[r * RS + i];
  }
}

// ------------------------------------------------------------------ y-fwd
template <typename T, int L>
__global__ void __launch_bounds__(256) k_yfwd(HotDev h) {
  using T2 = typename CT<T>::T2;
  const int TW = h.twy;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + L * TW;
  const int b = blockIdx.z;
  const int z = h.zplanes[blockIdx.y];
  const int x0 = blockIdx.x * TW;
  const int W = 8 * h.Nx;          // row width in complex elements (2Nx * 4)
  const int Ny = h.Ny;
  load_tw(tw, (const T2*)h.twy_tab, L);
  const T2* __restrict__ in = (const T2*)h.bufA + b * h.sA + (int64_t)z * Ny * W + x0;
  for (int i = threadIdx.x; i < Ny * TW; i += blockDim.x) {
    const int y = i / TW, w = i - y * TW;
    cp_async(b0 + i, in + (int64_t)y * W + w);
  }
  for (int i = Ny * TW + threadIdx.x; i < L * TW; i += blockDim.x) b0[i] = mk<T2>(0, 0);
  cp_async_wait_all();
  __syncthreads();
  T2* src = b0;
  T2* dst = b1;
  smem_fft<T2, L, false>(src, dst, TW, tw, ColAddr{TW});
  T2* __restrict__ out = (T2*)h.bufB + b * h.sB + (int64_t)z * L * W + x0;
  for (int i = threadIdx.x; i < L * TW; i += blockDim.x) {
    const int y = i / TW, w = i - y * TW;
    out[(int64_t)y * W + w] = src[i];
  }
}

// ------------------------------------------------------------------ z fwd * H * z inv
template <typename T, int L>
__global__ void __launch_bounds__(256) k_zconv(HotDev h) {
  using T2 = typename CT<T>::T2;
  const int TW = h.twz;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + L * TW;
  const int b = blockIdx.z;
  const int ky = blockIdx.y;
  const int x0 = blockIdx.x * TW;
  const int W = 8 * h.Nx;
  const int Ny2 = 2 * h.Ny;
  const int64_t zs = (int64_t)Ny2 * W;   // z stride in bufB
  load_tw(tw, (const T2*)h.twz_tab, L);
  if (h.nzocc < h.Nz)
    for (int i = threadIdx.x; i < L * TW; i += blockDim.x) b0[i] = mk<T2>(0, 0);
  else
    for (int i = h.Nz * TW + threadIdx.x; i < L * TW; i += blockDim.x) b0[i] = mk<T2>(0, 0);
  __syncthreads();
  T2* __restrict__ g = (T2*)h.bufB + b * h.sB + (int64_t)ky * W + x0;
  for (int i = threadIdx.x; i < h.nzocc * TW; i += blockDim.x) {
    const int zi = i / TW, w = i - zi * TW;
    const int z = h.zplanes[zi];
    cp_async(b0 + z * TW + w, g + z * zs + w);
  }
  cp_async_wait_all();
  __syncthreads();
  T2* src = b0;
  T2* dst = b1;
  smem_fft<T2, L, false>(src, dst, TW, tw, ColAddr{TW});
  {  // spectrum multiply (octant [ky][kz][kx], 1/M folded into H)
    const int Nx = h.Nx, Ny = h.Ny, Nz = h.Nz;
    const int kyf = ky <= Ny ? ky : Ny2 - ky;
    const T2* __restrict__ H = (const T2*)h.Hoct + b * h.sH + (int64_t)kyf * (Nz + 1) * (Nx + 1);
    for (int i = threadIdx.x; i < L * TW; i += blockDim.x) {
      const int kz = i / TW, w = i - kz * TW;
      const int kx = (x0 + w) >> 2;
      const int kxf = kx <= Nx ? kx : 2 * Nx - kx;
      const int kzf = kz <= Nz ? kz : 2 * Nz - kz;
      src[i] = cmul(src[i], H[(int64_t)kzf * (Nx + 1) + kxf]);
    }
  }
  __syncthreads();
  smem_fft<T2, L, true>(src, dst, TW, tw, ColAddr{TW});
  for (int i = threadIdx.x; i < h.nzocc * TW; i += blockDim.x) {
    const int zi = i / TW, w = i - zi * TW;
    const int z = h.zplanes[zi];
    g[z * zs + w] = src[z * TW + w];
  }
}

// ------------------------------------------------------------------ y-inv
template <typename T, int L>
__global__ void __launch_bounds__(256) k_yinv(HotDev h) {
  using T2 = typename CT<T>::T2;
  const int TW = h.twy;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + L * TW;
  const int b = blockIdx.z;
  const int z = h.zplanes[blockIdx.y];
  const int x0 = blockIdx.x * TW;
  const int W = 8 * h.Nx;
  const int Ny = h.Ny;
  load_tw(tw, (const T2*)h.twy_tab, L);
  const T2* __restrict__ in = (const T2*)h.bufB + b * h.sB + (int64_t)z * L * W + x0;
  for (int i = threadIdx.x; i < L * TW; i += blockDim.x) {
    const int y = i / TW, w = i - y * TW;
    cp_async(b0 + i, in + (int64_t)y * W + w);
  }
  cp_async_wait_all();
  __syncthreads();
  T2* src = b0;
  T2* dst = b1;
  smem_fft<T2, L, true>(src, dst, TW, tw, ColAddr{TW});
  T2* __restrict__ out = (T2*)h.bufC + b * h.sA + (int64_t)z * Ny * W + x0;
  const uint8_t* occ = h.line_occ + (int64_t)z * Ny;
  for (int i = threadIdx.x; i < Ny * TW; i += blockDim.x) {
    const int y = i / TW, w = i - y * TW;
    if (occ[y]) out[(int64_t)y * W + w] = src[i];
  }
}

// ------------------------------------------------------------------ x-inv
template <typename T, int L>
__global__ void __launch_bounds__(256) k_xinv(HotDev h) {
  using T2 = typename CT<T>::T2;
  constexpr int ROWS = rows_x<T>(L);
  constexpr int RS = (L + 1) * 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + ROWS * RS;
  const int b = blockIdx.y;
  const int l0 = blockIdx.x * ROWS;
  const int nrows = min(ROWS, h.nlines - l0);
  load_tw(tw, (const T2*)h.twx, L);
  const T2* __restrict__ in = (const T2*)h.bufC + b * h.sA;
  for (int i = threadIdx.x; i < nrows * L * 4; i += blockDim.x) {
    const int r = i / (L * 4), e = i - r * (L * 4);
    cp_async(b0 + r * RS + e, in + (int64_t)h.line_id[l0 + r] * L * 4 + e);
  }
  cp_async_wait_all();
  __syncthreads();
  T2* src = b0;
  T2* dst = b1;
  smem_fft<T2, L, true>(src, dst, nrows * 4, tw, RowAddr<L>{});
  T2* __restrict__ out = (T2*)h.phi + b * h.sP;
  const int Nx = h.Nx;
  for (int r = 0; r < nrows; ++r) {
    const int64_t base = (int64_t)h.line_id[l0 + r] * Nx * 4;
    for (int i = threadIdx.x; i < Nx * 4; i += blockDim.x) out[base + i] = src[r * RS + i];
  }
}

// ------------------------------------------------------------------ S4 + S5
template <typename T2> __device__ __forceinline__ T2 warp_sum(T2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

template <typename T, int BB>
__global__ void __launch_bounds__(256) k_interp_near(HotDev h, const typename CT<T>::T2* __restrict__ x,
                                                     typename CT<T>::T2* __restrict__ y0,
                                                     typename CT<T>::T2* __restrict__ y1, Combine cb) {
  using T2 = typename CT<T>::T2;
  using T4 = typename CT<T>::T4;
  const int lane = threadIdx.x & 31;
  const int m = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (m >= h.nb) return;
  const int B = cb.B;
  T2 aA[BB], aR[BB];
#pragma unroll
  for (int b = 0; b < BB; ++b) {
    aA[b] = mk<T2>(0, 0);
    aR[b] = mk<T2>(0, 0);
  }
  for (int sl = lane; sl < h.p3; sl += 32) {
    const int p = h.p;
    const int i = sl % p, j = (sl / p) % p, k = sl / (p * p);
    const int64_t lin = (int64_t)h.rwg_base[m] + i + (int64_t)h.Nx * (j + (int64_t)h.Ny * k);
    const T4 w = ((const T4*)h.lam)[(int64_t)m * h.p3 + sl];
#pragma unroll
    for (int b = 0; b < BB; ++b) {
      if (b < B) {
        const T2* ph = (const T2*)h.phi + b * h.sP + lin * 4;
        const T2 p0 = ph[0], p1 = ph[1], p2 = ph[2], p3 = ph[3];
        aA[b].x += w.x * p0.x + w.y * p1.x + w.z * p2.x;
        aA[b].y += w.x * p0.y + w.y * p1.y + w.z * p2.y;
        aR[b].x += w.w * p3.x;
        aR[b].y += w.w * p3.y;
      }
    }
  }
  const T2* __restrict__ cv = (const T2*)h.cval;
  const int kb = h.rowptr[m], ke = h.rowptr[m + 1];
  // x for the near rows: batch-interleaved xt[n * BB + b] (BB > 1) or x itself
  for (int kk = kb + lane; kk < ke; kk += 32) {
    const int n = h.col[kk];
    const T2 c = cv[kk];
    const T2* __restrict__ xr = x + (int64_t)n * BB;
    T2 xv[BB];
#pragma unroll
    for (int b = 0; b < BB; ++b) xv[b] = xr[b];
#pragma unroll
    for (int b = 0; b < BB; ++b) {
      aA[b].x += c.x * xv[b].x; aA[b].y += c.x * xv[b].y;
      aR[b].x += c.y * xv[b].x; aR[b].y += c.y * xv[b].y;
    }
  }
  using R = decltype(T2::x);
#pragma unroll
  for (int b = 0; b < BB; ++b) {
    if (b < B) {
      const T2 sA = warp_sum(aA[b]);
      const T2 sR = warp_sum(aR[b]);
      if (lane == 0) {
        if (cb.mode == 0) {
          const R al = (R)cb.alpha_im[b], be = (R)cb.beta[b];
          const R ux = sA.x - be * sR.x, uy = sA.y - be * sR.y;
          y0[b * cb.ystride + m] = mk<T2>(-al * uy, al * ux);   // (j alpha) * u
        } else {
          if (y0) y0[b * cb.ystride + m] = sA;
          if (y1) y1[b * cb.ystride + m] = mk<T2>(-sR.x, -sR.y);
        }
      }
    }
  }
}

// ------------------------------------------------------------------ dispatch
template <class K> void set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    AIMX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

template <typename T>
void run_gather(const HotDev& h, const void* x, int64_t xstride, int B, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const int per = 256 / h.G;
  dim3 g((unsigned)((h.nocc + per - 1) / per), (unsigned)B);
  switch (h.G) {
    case 4: k_gather<T, 4><<<g, 256, 0, s>>>(h, (const T2*)x, xstride); break;
    case 8: k_gather<T, 8><<<g, 256, 0, s>>>(h, (const T2*)x, xstride); break;
    case 16: k_gather<T, 16><<<g, 256, 0, s>>>(h, (const T2*)x, xstride); break;
    default: k_gather<T, 32><<<g, 256, 0, s>>>(h, (const T2*)x, xstride); break;
  }
  AIMX_CHECK_LAUNCH();
}

template <typename T, int L>
void run_x(const HotDev& h, bool inv, int B, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  constexpr int ROWS = rows_x<T>(L);
  const size_t sm = sizeof(T2) * (L + 2 * ROWS * (L + 1) * 4);
  dim3 g((unsigned)((h.nlines + ROWS - 1) / ROWS), (unsigned)B);
  if (!inv) {
    set_smem(k_xfwd<T, L>, sm);
    k_xfwd<T, L><<<g, 256, sm, s>>>(h);
  } else {
    set_smem(k_xinv<T, L>, sm);
    k_xinv<T, L><<<g, 256, sm, s>>>(h);
  }
  AIMX_CHECK_LAUNCH();
}

template <typename T, int L>
void run_y(const HotDev& h, bool inv, int B, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const size_t sm = sizeof(T2) * (L + 2 * (size_t)L * h.twy);
  dim3 g((unsigned)(8 * h.Nx / h.twy), (unsigned)h.nzocc, (unsigned)B);
  if (!inv) {
    set_smem(k_yfwd<T, L>, sm);
    k_yfwd<T, L><<<g, 256, sm, s>>>(h);
  } else {
    set_smem(k_yinv<T, L>, sm);
    k_yinv<T, L><<<g, 256, sm, s>>>(h);
  }
  AIMX_CHECK_LAUNCH();
}

template <typename T, int L>
void run_z(const HotDev& h, int B, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const size_t sm = sizeof(T2) * (L + 2 * (size_t)L * h.twz);
  set_smem(k_zconv<T, L>, sm);
  dim3 g((unsigned)(8 * h.Nx / h.twz), (unsigned)(2 * h.Ny), (unsigned)B);
  k_zconv<T, L><<<g, 256, sm, s>>>(h);
  AIMX_CHECK_LAUNCH();
}

// xt[n * BB + b] = x[b * xstride + n] (zero for b >= B)
template <typename T>
__global__ void k_interleave(int nb, int B, int BB, const typename CT<T>::T2* __restrict__ x,
                             int64_t xstride, typename CT<T>::T2* __restrict__ xt) {
  using T2 = typename CT<T>::T2;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)nb * BB) return;
  const int n = (int)(i / BB), b = (int)(i - (int64_t)n * BB);
  xt[i] = b < B ? x[b * xstride + n] : mk<T2>(0, 0);
}

template <typename T>
void run_interp(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const unsigned g = (unsigned)(((int64_t)h.nb * 32 + 255) / 256);
  const T2* xx = (const T2*)x;
  if (c.B > 1) {
    const int BB = c.B <= 2 ? 2 : (c.B <= 4 ? 4 : (c.B <= 8 ? 8 : 16));
    const int64_t n = (int64_t)h.nb * BB;
    k_interleave<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h.nb, c.B, BB, xx, c.xstride,
                                                                (T2*)h.xt);
    AIMX_CHECK_LAUNCH();
    xx = (const T2*)h.xt;
  }
  if (c.B <= 1) k_interp_near<T, 1><<<g, 256, 0, s>>>(h, xx, (T2*)y0, (T2*)y1, c);
  else if (c.B <= 2) k_interp_near<T, 2><<<g, 256, 0, s>>>(h, xx, (T2*)y0, (T2*)y1, c);
  else if (c.B <= 4) k_interp_near<T, 4><<<g, 256, 0, s>>>(h, xx, (T2*)y0, (T2*)y1, c);
  else if (c.B <= 8) k_interp_near<T, 8><<<g, 256, 0, s>>>(h, xx, (T2*)y0, (T2*)y1, c);
  else k_interp_near<T, 16><<<g, 256, 0, s>>>(h, xx, (T2*)y0, (T2*)y1, c);
  AIMX_CHECK_LAUNCH();
}

template <typename T>
void hot_matvec(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s,
                Profiler* prof) {
  if (c.B < 1 || c.B > h.batch || c.B > kMaxBatch) throw Error(AIMX_E_INTERNAL, "bad batch");
  const int Lx = 2 * h.Nx, Ly = 2 * h.Ny, Lz = 2 * h.Nz, B = c.B;
  {
    StageScope sc(prof, 1, s);
    run_gather<T>(h, x, c.xstride, B, s);
    AIMX_SWITCH_L(Lx, (run_x<T, L>(h, false, B, s)));
  }
  { StageScope sc(prof, 2, s); AIMX_SWITCH_L(Ly, (run_y<T, L>(h, false, B, s))); }
  { StageScope sc(prof, 3, s); AIMX_SWITCH_L(Lz, (run_z<T, L>(h, B, s))); }
  { StageScope sc(prof, 4, s); AIMX_SWITCH_L(Ly, (run_y<T, L>(h, true, B, s))); }
  { StageScope sc(prof, 5, s); AIMX_SWITCH_L(Lx, (run_x<T, L>(h, true, B, s))); }
  { StageScope sc(prof, 6, s); run_interp<T>(h, x, y0, y1, c, s); }
}

}  // namespace

bool fft_length_supported(int L) { return L >= 8 && L <= 1024 && (L & (L - 1)) == 0; }

// Tile width (complex elements per row segment) of the strided y / z passes:
// about 4096 (fp32) / 2048 (fp64) elements per CTA, at least one 32-byte
// sector per row, at most the row width 8 N_x.
int pick_tile(int L, int rowwidth, bool f32) {
  int t = (f32 ? 4096 : 2048) / L;
  const int lo = f32 ? 4 : 2;
  if (t < lo) t = lo;
  if (t > 512) t = 512;
  if (t > rowwidth) t = rowwidth;
  return t;
}

void hot_matvec_f32(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c,
                    cudaStream_t s, Profiler* prof) {
  hot_matvec<float>(h, x, y0, y1, c, s, prof);
}
void hot_matvec_f64(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c,
                    cudaStream_t s, Profiler* prof) {
  hot_matvec<double>(h, x, y0, y1, c, s, prof);
}

cudaEvent_t Profiler::get() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  AIMX_CUDA(cudaEventCreate(&e));
  return e;
}
void Profiler::begin(int stage, cudaStream_t s, cudaEvent_t& a) {
  (void)stage;
  a = get();
  AIMX_CUDA(cudaEventRecord(a, s));
}
void Profiler::end(int stage, cudaStream_t s, cudaEvent_t a) {
  cudaEvent_t b = get();
  AIMX_CUDA(cudaEventRecord(b, s));
  pending.push_back({stage, a, b});
  if (pending.size() > 16384) collect();
}
void Profiler::collect() {
  for (auto& r : pending) {
    AIMX_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    AIMX_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.stage] += t;
    n[r.stage] += 1;
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  pending.clear();
}
Profiler::~Profiler() {
  for (auto& r : pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : pool) cudaEventDestroy(e);
}

}  // namespace aimx
