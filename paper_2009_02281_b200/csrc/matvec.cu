// The AIMx hot path on the B200 (S2-S5), one kernel per stage:
//
//   k_proj_xfft   S2 + first pass of S3: gather the grid sources of every
//                 occupied x-line from the transposed (node-major) projection
//                 CSR -- no atomics -- and do the zero-padded forward FFT along x.
//   k_yfwd        forward FFT along y (input rows y < N_y, zero padded)
//   k_zconv       forward FFT along z, times the spectrum H_hat (octant,
//                 already scaled by 1/M), inverse FFT along z, cropped to z < N_z
//   k_yinv        inverse FFT along y, cropped to y < N_y (occupied lines only)
//   k_xinv        inverse FFT along x, cropped to x < N_x -> potentials phi
//   k_interp_near S4 + S5: warp per RWG (testing function): interpolation
//                 W = P^T of the 4 potentials on its (n+1)^3 stencil, plus the
//                 near-region row of C = L_s,NR - L_s,P, plus the EFIE combine
//                 y = -j w mu0 (y^A - k0^-2 y^rho).
//
// P:198-200 (W H P, "accelerated with FFTs", applied on the entire grid);
// eq:LAIMx P:283; eq:EFIEAIMx P:288.  Grid data are complex, 4 channels
// (x, y, z, rho) innermost: element ((z * Ny' + y) * Nx' + x) * 4 + c.
// Pruning (exact, reading R12): lines/planes with no occupied node are never
// transformed; their data are identically zero and are never read as input.
//
// The FFTs are shared-memory Stockham radix-8/4/2 passes over tiles of lines
// (ping-pong buffers, twiddle table in shared memory).
#include <algorithm>

#include "aimx_internal.h"

namespace aimx {

namespace {

template <typename T> struct CT;
template <> struct CT<float> { using T2 = float2; using T4 = float4; };
template <> struct CT<double> { using T2 = double2; using T4 = double4; };

template <typename T2> __device__ __forceinline__ T2 mk(decltype(T2::x) a, decltype(T2::x) b) {
  T2 r; r.x = a; r.y = b; return r;
}
template <typename T2> __device__ __forceinline__ T2 cadd(T2 a, T2 b) { return mk<T2>(a.x + b.x, a.y + b.y); }
template <typename T2> __device__ __forceinline__ T2 csub(T2 a, T2 b) { return mk<T2>(a.x - b.x, a.y - b.y); }
template <typename T2> __device__ __forceinline__ T2 cmul(T2 a, T2 b) {
  return mk<T2>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// multiply by -j (forward) or +j (inverse)
template <typename T2, bool INV> __device__ __forceinline__ T2 mulj(T2 a) {
  return INV ? mk<T2>(-a.y, a.x) : mk<T2>(a.y, -a.x);
}

template <typename T2, bool INV> __device__ __forceinline__ void dft2(T2* v) {
  T2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}
template <typename T2, bool INV> __device__ __forceinline__ void dft4(T2& v0, T2& v1, T2& v2, T2& v3) {
  T2 t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = mulj<T2, INV>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v2 = csub(t0, t2);
  v1 = cadd(t1, t3);
  v3 = csub(t1, t3);
}
template <typename T2, bool INV> __device__ __forceinline__ void dft8(T2* v) {
  using R = decltype(T2::x);
  T2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  T2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<T2, INV>(e0, e1, e2, e3);
  dft4<T2, INV>(o0, o1, o2, o3);
  const R s = (R)0.70710678118654752440;
  // W8^1 = (1 -+ j)/sqrt2, W8^2 = -+j, W8^3 = (-1 -+ j)/sqrt2
  T2 w1 = INV ? mk<T2>(s * (o1.x - o1.y), s * (o1.x + o1.y)) : mk<T2>(s * (o1.x + o1.y), s * (o1.y - o1.x));
  T2 w2 = mulj<T2, INV>(o2);
  T2 w3 = INV ? mk<T2>(-s * (o3.x + o3.y), s * (o3.x - o3.y)) : mk<T2>(s * (o3.y - o3.x), -s * (o3.x + o3.y));
  v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
  v[1] = cadd(e1, w1); v[5] = csub(e1, w1);
  v[2] = cadd(e2, w2); v[6] = csub(e2, w2);
  v[3] = cadd(e3, w3); v[7] = csub(e3, w3);
}
template <typename T2, int R, bool INV> __device__ __forceinline__ void dft(T2* v) {
  if constexpr (R == 2) dft2<T2, INV>(v);
  else if constexpr (R == 4) dft4<T2, INV>(v[0], v[1], v[2], v[3]);
  else dft8<T2, INV>(v);
}

// Column layout: element (line, idx) at idx * TW + line.
template <int TW> struct ColAddr {
  __device__ __forceinline__ int operator()(int line, int idx) const { return idx * TW + line; }
};
// Row layout with 4 channels innermost, rows padded by one node (bank spread).
template <int L> struct RowAddr {
  __device__ __forceinline__ int operator()(int line, int idx) const {
    return (line >> 2) * ((L + 1) * 4) + idx * 4 + (line & 3);
  }
};

// One Stockham stage: src -> dst.
template <typename T2, int L, int R, int NS, bool INV, class Addr>
__device__ __forceinline__ void fft_stage(const T2* __restrict__ src, T2* __restrict__ dst, int nlines,
                                          const T2* __restrict__ tw, Addr addr) {
  constexpr int NB = L / R;
  const int total = nlines * NB;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int line = t % nlines;
    const int j = t / nlines;
    const int k = j % NS;
    T2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[addr(line, j + r * NB)];
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        T2 w = tw[(r * k * (L / (NS * R))) & (L - 1)];
        if (INV) w.y = -w.y;
        v[r] = cmul(v[r], w);
      }
    }
    dft<T2, R, INV>(v);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[addr(line, base + r * NS)] = v[r];
  }
}

template <typename T2, int L, bool INV, int NS, class Addr>
__device__ __forceinline__ void fft_stages(T2*& src, T2*& dst, int nlines, const T2* tw, Addr addr) {
  if constexpr (NS < L) {
    constexpr int REM = L / NS;
    constexpr int R = (REM % 8 == 0) ? 8 : ((REM % 4 == 0) ? 4 : 2);
    fft_stage<T2, L, R, NS, INV>(src, dst, nlines, tw, addr);
    __syncthreads();
    T2* t = src;
    src = dst;
    dst = t;
    fft_stages<T2, L, INV, NS * R>(src, dst, nlines, tw, addr);
  }
}

// Result ends in `src` (swapped as stages proceed).
template <typename T2, int L, bool INV, class Addr>
__device__ __forceinline__ void smem_fft(T2*& src, T2*& dst, int nlines, const T2* tw, Addr addr) {
  fft_stages<T2, L, INV, 1>(src, dst, nlines, tw, addr);
}

template <typename T> constexpr int tile_w(int L) {
  // complex elements per row segment for the strided (y, z) passes
  int t = (int)(sizeof(T) == 4 ? 4096 : 2048) / L;
  int lo = sizeof(T) == 4 ? 4 : 2;
  return t < lo ? lo : (t > 64 ? 64 : t);
}
template <typename T> constexpr int rows_x(int L) {
  int r = (sizeof(T) == 4 ? 4096 : 2048) / (4 * L);
  return r < 1 ? 1 : (r > 32 ? 32 : r);
}

template <typename T2>
__device__ __forceinline__ void load_tw(T2* s_tw, const T2* __restrict__ g_tw, int L) {
  for (int i = threadIdx.x; i < L; i += blockDim.x) s_tw[i] = g_tw[i];
}

// ------------------------------------------------------------------ S2 + x-fwd
template <typename T, int L>
__global__ void __launch_bounds__(256) k_proj_xfft(HotDev h, const typename CT<T>::T2* __restrict__ x) {
  using T2 = typename CT<T>::T2;
  using T4 = typename CT<T>::T4;
  constexpr int ROWS = rows_x<T>(L);
  constexpr int RS = (L + 1) * 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + ROWS * RS;
  const int l0 = blockIdx.x * ROWS;
  const int nrows = min(ROWS, h.nlines - l0);
  load_tw(tw, (const T2*)h.twx, L);
  for (int i = threadIdx.x; i < ROWS * RS; i += blockDim.x) b0[i] = mk<T2>(0, 0);
  __syncthreads();
  const int q0 = h.line_ptr[l0], q1 = h.line_ptr[l0 + nrows];
  const T4* __restrict__ ew = (const T4*)h.ent_w;
  for (int q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    // row of node q: largest r with line_ptr[l0 + r] <= q
    int lo = 0, hi = nrows - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (h.line_ptr[l0 + mid] <= q) lo = mid; else hi = mid - 1;
    }
    const int xx = h.node_lin[q] % h.Nx;
    T2 a0 = mk<T2>(0, 0), a1 = a0, a2 = a0, a3 = a0;
    for (int e = h.node_ptr[q]; e < h.node_ptr[q + 1]; ++e) {
      const T4 w = ew[e];
      const T2 xv = x[h.ent_rwg[e]];
      a0.x += w.x * xv.x; a0.y += w.x * xv.y;
      a1.x += w.y * xv.x; a1.y += w.y * xv.y;
      a2.x += w.z * xv.x; a2.y += w.z * xv.y;
      a3.x += w.w * xv.x; a3.y += w.w * xv.y;
    }
    T2* dst = b0 + lo * RS + xx * 4;
    dst[0] = a0; dst[1] = a1; dst[2] = a2; dst[3] = a3;
  }
  __syncthreads();
  T2* src = b0;
  T2* dst = b1;
  smem_fft<T2, L, false>(src, dst, nrows * 4, tw, RowAddr<L>{});
  T2* __restrict__ out = (T2*)h.bufA;
  for (int r = 0; r < nrows; ++r) {
    const int64_t base = (int64_t)h.line_id[l0 + r] * L * 4;
    for (int i = threadIdx.x; i < L * 4; i += blockDim.x) out[base + i] = src[r * RS + i];
  }
}

// ------------------------------------------------------------------ y-fwd
template <typename T, int L>
__global__ void __launch_bounds__(256) k_yfwd(HotDev h) {
  using T2 = typename CT<T>::T2;
  constexpr int TW = tile_w<T>(L);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + L * TW;
  const int z = h.zplanes[blockIdx.y];
  const int x0 = blockIdx.x * TW;
  const int W = 8 * h.Nx;          // row width in complex elements (2Nx * 4)
  const int Ny = h.Ny;
  load_tw(tw, (const T2*)h.twy, L);
  const T2* __restrict__ in = (const T2*)h.bufA + (int64_t)z * Ny * W + x0;
  for (int i = threadIdx.x; i < L * TW; i += blockDim.x) {
    const int y = i / TW, w = i % TW;
    b0[i] = (y < Ny) ? in[(int64_t)y * W + w] : mk<T2>(0, 0);
  }
  __syncthreads();
  T2* src = b0;
  T2* dst = b1;
  smem_fft<T2, L, false>(src, dst, TW, tw, ColAddr<TW>{});
  T2* __restrict__ out = (T2*)h.bufB + (int64_t)z * L * W + x0;
  for (int i = threadIdx.x; i < L * TW; i += blockDim.x) {
    const int y = i / TW, w = i % TW;
    out[(int64_t)y * W + w] = src[i];
  }
}

// ------------------------------------------------------------------ z fwd * H * z inv
template <typename T, int L>
__global__ void __launch_bounds__(256) k_zconv(HotDev h) {
  using T2 = typename CT<T>::T2;
  constexpr int TW = tile_w<T>(L);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + L * TW;
  const int ky = blockIdx.y;
  const int x0 = blockIdx.x * TW;
  const int W = 8 * h.Nx;
  const int Ny2 = 2 * h.Ny;
  const int64_t zs = (int64_t)Ny2 * W;   // z stride in bufB
  load_tw(tw, (const T2*)h.twz, L);
  for (int i = threadIdx.x; i < L * TW; i += blockDim.x) b0[i] = mk<T2>(0, 0);
  __syncthreads();
  T2* __restrict__ g = (T2*)h.bufB + (int64_t)ky * W + x0;
  for (int i = threadIdx.x; i < h.nzocc * TW; i += blockDim.x) {
    const int z = h.zplanes[i / TW], w = i % TW;
    b0[z * TW + w] = g[z * zs + w];
  }
  __syncthreads();
  T2* src = b0;
  T2* dst = b1;
  smem_fft<T2, L, false>(src, dst, TW, tw, ColAddr<TW>{});
  // spectrum multiply (octant index, 1/M folded into H)
  {
    const int Nx = h.Nx, Ny = h.Ny, Nz = h.Nz;
    const int kyf = ky <= Ny ? ky : Ny2 - ky;
    const T2* __restrict__ H = (const T2*)h.Hoct;
    for (int i = threadIdx.x; i < L * TW; i += blockDim.x) {
      const int kz = i / TW, w = i % TW;
      const int kx = (x0 + w) >> 2;
      const int kxf = kx <= Nx ? kx : 2 * Nx - kx;
      const int kzf = kz <= Nz ? kz : 2 * Nz - kz;
      const T2 hv = H[((int64_t)kyf * (Nx + 1) + kxf) * (Nz + 1) + kzf];
      src[i] = cmul(src[i], hv);
    }
  }
  __syncthreads();
  smem_fft<T2, L, true>(src, dst, TW, tw, ColAddr<TW>{});
  for (int i = threadIdx.x; i < h.nzocc * TW; i += blockDim.x) {
    const int z = h.zplanes[i / TW], w = i % TW;
    g[z * zs + w] = src[z * TW + w];
  }
}

// ------------------------------------------------------------------ y-inv
template <typename T, int L>
__global__ void __launch_bounds__(256) k_yinv(HotDev h) {
  using T2 = typename CT<T>::T2;
  constexpr int TW = tile_w<T>(L);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* b0 = tw + L;
  T2* b1 = b0 + L * TW;
  const int z = h.zplanes[blockIdx.y];
  const int x0 = blockIdx.x * TW;
  const int W = 8 * h.Nx;
  const int Ny = h.Ny;
  load_tw(tw, (const T2*)h.twy, L);
  const T2* __restrict__ in = (const T2*)h.bufB + (int64_t)z * L * W + x0;
  for (int i = threadIdx.x; i < L * TW; i += blockDim.x) {
    const int y = i / TW, w = i % TW;
    b0[i] = in[(int64_t)y * W + w];
  }
  __syncthreads();
  T2* src = b0;
  T2* dst = b1;
  smem_fft<T2, L, true>(src, dst, TW, tw, ColAddr<TW>{});
  T2* __restrict__ out = (T2*)h.bufC + (int64_t)z * Ny * W + x0;
  const uint8_t* occ = h.line_occ + (int64_t)z * Ny;
  for (int i = threadIdx.x; i < Ny * TW; i += blockDim.x) {
    const int y = i / TW, w = i % TW;
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
  const int l0 = blockIdx.x * ROWS;
  const int nrows = min(ROWS, h.nlines - l0);
  load_tw(tw, (const T2*)h.twx, L);
  const T2* __restrict__ in = (const T2*)h.bufC;
  for (int r = 0; r < nrows; ++r) {
    const int64_t base = (int64_t)h.line_id[l0 + r] * L * 4;
    for (int i = threadIdx.x; i < L * 4; i += blockDim.x) b0[r * RS + i] = in[base + i];
  }
  __syncthreads();
  T2* src = b0;
  T2* dst = b1;
  smem_fft<T2, L, true>(src, dst, nrows * 4, tw, RowAddr<L>{});
  T2* __restrict__ out = (T2*)h.phi;
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

template <typename T>
__global__ void __launch_bounds__(256) k_interp_near(HotDev h, const typename CT<T>::T2* __restrict__ x,
                                                     typename CT<T>::T2* __restrict__ y0,
                                                     typename CT<T>::T2* __restrict__ y1, Combine cb) {
  using T2 = typename CT<T>::T2;
  using T4 = typename CT<T>::T4;
  const int lane = threadIdx.x & 31;
  const int m = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (m >= h.nb) return;
  T2 aA = mk<T2>(0, 0), aR = mk<T2>(0, 0);
  for (int sl = lane; sl < h.p3; sl += 32) {
    const int p = h.p;
    const int i = sl % p, j = (sl / p) % p, k = sl / (p * p);
    const int64_t lin = (int64_t)h.rwg_base[m] + i + (int64_t)h.Nx * (j + (int64_t)h.Ny * k);
    const T2* ph = (const T2*)h.phi + lin * 4;
    const T4 w = ((const T4*)h.lam)[(int64_t)m * h.p3 + sl];
    const T2 p0 = ph[0], p1 = ph[1], p2 = ph[2], p3 = ph[3];
    aA.x += w.x * p0.x + w.y * p1.x + w.z * p2.x;
    aA.y += w.x * p0.y + w.y * p1.y + w.z * p2.y;
    aR.x += w.w * p3.x;
    aR.y += w.w * p3.y;
  }
  const T2* __restrict__ cv = (const T2*)h.cval;
  const int kb = h.rowptr[m], ke = h.rowptr[m + 1];
  for (int kk = kb + lane; kk < ke; kk += 32) {
    const int n = h.col[kk];
    const T2 c = cv[kk];
    const T2 xv = x[n];
    aA.x += c.x * xv.x; aA.y += c.x * xv.y;
    aR.x += c.y * xv.x; aR.y += c.y * xv.y;
  }
  aA = warp_sum(aA);
  aR = warp_sum(aR);
  if (lane == 0) {
    using R = decltype(T2::x);
    if (cb.mode == 0) {
      const R al = (R)cb.alpha_im, be = (R)cb.beta;
      const R ux = aA.x - be * aR.x, uy = aA.y - be * aR.y;
      y0[m] = mk<T2>(-al * uy, al * ux);   // (j alpha) * u
    } else {
      if (y0) y0[m] = aA;
      if (y1) y1[m] = mk<T2>(-aR.x, -aR.y);
    }
  }
}

// ------------------------------------------------------------------ dispatch
template <typename T, int L> size_t smem_rows() {
  return sizeof(typename CT<T>::T2) * (L + 2 * rows_x<T>(L) * (L + 1) * 4);
}
template <typename T, int L> size_t smem_cols() {
  return sizeof(typename CT<T>::T2) * (L + 2 * L * tile_w<T>(L));
}

template <class K> void set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) AIMX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

template <typename T, int L>
void run_x_fwd(const HotDev& h, const void* x, cudaStream_t s) {
  constexpr int ROWS = rows_x<T>(L);
  size_t sm = smem_rows<T, L>();
  set_smem(k_proj_xfft<T, L>, sm);
  unsigned g = (unsigned)((h.nlines + ROWS - 1) / ROWS);
  k_proj_xfft<T, L><<<g, 256, sm, s>>>(h, (const typename CT<T>::T2*)x);
  AIMX_CHECK_LAUNCH();
}
template <typename T, int L>
void run_x_inv(const HotDev& h, cudaStream_t s) {
  constexpr int ROWS = rows_x<T>(L);
  size_t sm = smem_rows<T, L>();
  set_smem(k_xinv<T, L>, sm);
  unsigned g = (unsigned)((h.nlines + ROWS - 1) / ROWS);
  k_xinv<T, L><<<g, 256, sm, s>>>(h);
  AIMX_CHECK_LAUNCH();
}
template <typename T, int L>
void run_y(const HotDev& h, bool inv, cudaStream_t s) {
  constexpr int TW = tile_w<T>(L);
  size_t sm = smem_cols<T, L>();
  dim3 g((unsigned)(8 * h.Nx / TW), (unsigned)h.nzocc);
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
void run_z(const HotDev& h, cudaStream_t s) {
  constexpr int TW = tile_w<T>(L);
  size_t sm = smem_cols<T, L>();
  set_smem(k_zconv<T, L>, sm);
  dim3 g((unsigned)(8 * h.Nx / TW), (unsigned)(2 * h.Ny));
  k_zconv<T, L><<<g, 256, sm, s>>>(h);
  AIMX_CHECK_LAUNCH();
}

#define AIMX_SWITCH_L(Lv, CALL)                     \
  switch (Lv) {                                     \
    case 8: { constexpr int L = 8; CALL; } break;     \
    case 16: { constexpr int L = 16; CALL; } break;   \
    case 32: { constexpr int L = 32; CALL; } break;   \
    case 64: { constexpr int L = 64; CALL; } break;   \
    case 128: { constexpr int L = 128; CALL; } break; \
    case 256: { constexpr int L = 256; CALL; } break; \
    case 512: { constexpr int L = 512; CALL; } break; \
    case 1024: { constexpr int L = 1024; CALL; } break; \
    default: throw Error(AIMX_E_UNSUPPORTED, "FFT length not compiled"); \
  }

template <typename T>
void hot_matvec(const HotDev& h, const void* x, void* y0, void* y1, Combine c, cudaStream_t s,
                Profiler* prof) {
  using T2 = typename CT<T>::T2;
  const int Lx = 2 * h.Nx, Ly = 2 * h.Ny, Lz = 2 * h.Nz;
  { StageScope sc(prof, 1, s); AIMX_SWITCH_L(Lx, (run_x_fwd<T, L>(h, x, s))); }
  { StageScope sc(prof, 2, s); AIMX_SWITCH_L(Ly, (run_y<T, L>(h, false, s))); }
  { StageScope sc(prof, 3, s); AIMX_SWITCH_L(Lz, (run_z<T, L>(h, s))); }
  { StageScope sc(prof, 4, s); AIMX_SWITCH_L(Ly, (run_y<T, L>(h, true, s))); }
  { StageScope sc(prof, 5, s); AIMX_SWITCH_L(Lx, (run_x_inv<T, L>(h, s))); }
  {
    StageScope sc(prof, 6, s);
    unsigned g = (unsigned)(((int64_t)h.nb * 32 + 255) / 256);
    k_interp_near<T><<<g, 256, 0, s>>>(h, (const T2*)x, (T2*)y0, (T2*)y1, c);
    AIMX_CHECK_LAUNCH();
  }
}

}  // namespace

bool fft_length_supported(int L) {
  return L >= 8 && L <= 1024 && (L & (L - 1)) == 0;
}

void hot_matvec_f32(const HotDev& h, const void* x, void* y0, void* y1, Combine c, cudaStream_t s,
                    Profiler* prof) {
  hot_matvec<float>(h, x, y0, y1, c, s, prof);
}
void hot_matvec_f64(const HotDev& h, const void* x, void* y0, void* y1, Combine c, cudaStream_t s,
                    Profiler* prof) {
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
  for (auto& r : pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : pool) cudaEventDestroy(e);
}

}  // namespace aimx
