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
#include <type_traits>

#include "aimx_internal.h"
#include "fft.cuh"
#include "fft_reg.cuh"

namespace aimx {

namespace {

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

// S2 for BB right-hand sides at once (batch-interleaved xt[n * BB + b]):
// warp per occupied node, groups of BB/V lanes stride its entries (each entry's
// weights and RWG index read once for all columns), lanes cover columns.
template <typename T, int BB>
__global__ void __launch_bounds__(256) k_gather_b(HotDev h, const typename CT<T>::T2* __restrict__ xt,
                                                  int B) {
  using T2 = typename CT<T>::T2;
  using T4 = typename CT<T>::T4;
  constexpr int V = sizeof(T2) == 8 ? 2 : 1;
  constexpr int LG = BB / V, NG = 32 / LG;
  using VT = typename std::conditional<V == 2, float4, double2>::type;
  const int lane = threadIdx.x & 31;
  const int b0 = (lane % LG) * V, g = lane / LG;
  const int q = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (q >= h.nocc) return;
  T2 a[V][4];
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int c = 0; c < 4; ++c) a[v][c] = mk<T2>(0, 0);
  const T4* __restrict__ ew = (const T4*)h.ent_w;
  const int e0 = h.node_ptr[q], e1 = h.node_ptr[q + 1];
  for (int base = e0; base < e1; base += 32) {
    // 32 entries loaded coalesced, then handed to the groups by shuffles
    const int ee = base + lane;
    const bool ok = ee < e1;
    const int myr = ok ? h.ent_rwg[ee] : 0;
    const T4 myw = ok ? ew[ee] : T4{0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 32; j += NG) {
    const int src = j + g;
    if (base + j >= e1) break;
    T4 w;
    w.x = __shfl_sync(0xffffffffu, myw.x, src);
    w.y = __shfl_sync(0xffffffffu, myw.y, src);
    w.z = __shfl_sync(0xffffffffu, myw.z, src);
    w.w = __shfl_sync(0xffffffffu, myw.w, src);
    const int rr = __shfl_sync(0xffffffffu, myr, src);
    const VT u = *(const VT*)(xt + (int64_t)rr * BB + b0);
    T2 xv[V];
    if constexpr (V == 2) {
      xv[0] = mk<T2>(u.x, u.y);
      xv[1] = mk<T2>(u.z, u.w);
    } else {
      xv[0] = u;
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      a[v][0].x += w.x * xv[v].x; a[v][0].y += w.x * xv[v].y;
      a[v][1].x += w.y * xv[v].x; a[v][1].y += w.y * xv[v].y;
      a[v][2].x += w.z * xv[v].x; a[v][2].y += w.z * xv[v].y;
      a[v][3].x += w.w * xv[v].x; a[v][3].y += w.w * xv[v].y;
    }
    }
  }
#pragma unroll
  for (int o = LG; o < 32; o <<= 1)
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        a[v][c].x += __shfl_xor_sync(0xffffffffu, a[v][c].x, o);
        a[v][c].y += __shfl_xor_sync(0xffffffffu, a[v][c].y, o);
      }
  if (g == 0) {
    const int64_t off = ((int64_t)h.node_line[q] * h.Nx + h.node_lin[q] % h.Nx) * 4;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int b = b0 + v;
      if (b < B) {
        T2* dst = (T2*)h.S + b * h.sS + off;
        dst[0] = a[v][0]; dst[1] = a[v][1]; dst[2] = a[v][2]; dst[3] = a[v][3];
      }
    }
  }
}

// ------------------------------------------------------------------ FFT passes
// Register-resident two-level FFTs (fft_reg.cuh).  Threads are mapped
// line-fastest (line = tid % NL, t = tid / NL) so that a warp's loads and
// stores cover consecutive grid columns; the per-line exchange uses one block
// barrier per transform.
template <typename S, int L> struct PassGeom {
  static constexpr int R1 = Fac<L>::R1, R2 = Fac<L>::R2;
  using TL = TwoLevel<R1, R2>;
  static constexpr int T = TL::T, E = TL::E;
  // per-line exchange stride: bank-spread so that the lines and threads of a
  // warp hit distinct 8-byte slots (stride = 1 mod 16, or 4 mod 16 when a
  // warp holds 8 lines x 4 threads)
  static constexpr int XB = R1 > 1 ? ((TL::XB + 15) / 16) * 16 + (T == 32 ? 4 : 1) : 0;
  static constexpr size_t BYTES256 = sizeof(typename CT<S>::T2) * (size_t)(256 / T) * XB;
  static constexpr int NT = BYTES256 > 200 * 1024 ? 128 : 256;   // threads per CTA
  static constexpr int NL = NT / T;                               // lines per CTA
};

template <typename T2, int L>
__device__ __forceinline__ void fwd_fft(T2* v, T2* xb, const T2* tw, int t) {
  fft2<T2, Fac<L>::R1, Fac<L>::R2, false>(v, xb, tw, t);
}
// inverse of data in the forward's output distribution, back to the input one
template <typename T2, int L>
__device__ __forceinline__ void inv_fft_swapped(T2* v, T2* xb, const T2* tw, int t) {
  fft2<T2, Fac<L>::R2, Fac<L>::R1, true>(v, xb, tw, t);
}
// inverse of data loaded in the input distribution (output distribution after)
template <typename T2, int L>
__device__ __forceinline__ void inv_fft(T2* v, T2* xb, const T2* tw, int t) {
  fft2<T2, Fac<L>::R1, Fac<L>::R2, true>(v, xb, tw, t);
}

template <typename T, int L>
__device__ __forceinline__ void pass_prologue(typename CT<T>::T2*& tw, typename CT<T>::T2*& xb,
                                              const typename CT<T>::T2* __restrict__ gtw, int line) {
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  tw = reinterpret_cast<T2*>(smem_raw);
  xb = tw + L + line * G::XB;
  for (int i = threadIdx.x; i < L; i += blockDim.x) tw[i] = gtw[i];
  __syncthreads();
}

template <typename T, int L> constexpr size_t pass_smem() {
  using G = PassGeom<T, L>;
  return sizeof(typename CT<T>::T2) * (L + (size_t)G::NL * G::XB);
}

// ---- x forward: occupied lines of S (x < Nx, zero padded) -> bufA[line_id][kx][c]
template <typename T, int L>
__global__ void __launch_bounds__(256) k_xfwd(HotDev h) {
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  T2 *tw, *xb;
  pass_prologue<T, L>(tw, xb, (const T2*)h.twx, line);
  const int b = blockIdx.y;
  const int r = blockIdx.x * (G::NL / 4) + (line >> 2), c = line & 3;
  const bool act = r < h.nlines;
  const int Nx = h.Nx;
  const T2* __restrict__ in = (const T2*)h.S + b * h.sS + (int64_t)r * Nx * 4 + c;
  T2 v[G::E];
#pragma unroll
  for (int i = 0; i < G::E; ++i) {   // x < Nx = L/2  <=>  n2 < R2/2
    const int x = G::TL::in_index(t, i);
    v[i] = (act && i % G::R2 < G::R2 / 2) ? in[x * 4] : mk<T2>(0, 0);
  }
  fwd_fft<T2, L>(v, xb, tw, t);
  if (!act) return;
  T2* __restrict__ out = (T2*)h.bufA + b * h.sA + (int64_t)h.line_id[r] * L * 4 + c;
#pragma unroll
  for (int i = 0; i < G::E; ++i) out[TwoLevel<G::R2, G::R1>::in_index(t, i) * 4] = v[i];
}

// ---- x inverse: bufC[line_id][kx][c] -> phi[line][x < Nx][c]
template <typename T, int L>
__global__ void __launch_bounds__(256) k_xinv(HotDev h) {
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  T2 *tw, *xb;
  pass_prologue<T, L>(tw, xb, (const T2*)h.twx, line);
  const int b = blockIdx.y;
  const int r = blockIdx.x * (G::NL / 4) + (line >> 2), c = line & 3;
  const bool act = r < h.nlines;
  const int lid = act ? h.line_id[r] : 0;
  const T2* __restrict__ in = (const T2*)h.bufC + b * h.sA + (int64_t)lid * L * 4 + c;
  T2 v[G::E];
#pragma unroll
  for (int i = 0; i < G::E; ++i) v[i] = act ? in[G::TL::in_index(t, i) * 4] : mk<T2>(0, 0);
  inv_fft<T2, L>(v, xb, tw, t);
  if (!act) return;
  const int Nx = h.Nx;
  // phi layout [node][channel][slot] (slots = batch, complex)
  const int64_t ns = (int64_t)h.batch * 4;   // node stride
  T2* __restrict__ out = (T2*)h.phi + (int64_t)c * h.batch + b + (int64_t)lid * Nx * ns;
#pragma unroll
  for (int i = 0; i < G::E; ++i) {   // x < Nx  <=>  k1 < R1/2 in D(R2,R1)
    const int x = TwoLevel<G::R2, G::R1>::in_index(t, i);
    if (i % G::R1 < (G::R1 + 1) / 2 && x < Nx) out[x * ns] = v[i];
  }
}

// Column passes: CTA = NL lines = (rows per CTA) x (column tile CW).
struct ColTile {
  int w, rsub, CW, RPC;
};
template <typename T, int L> __device__ __forceinline__ ColTile col_tile(int line, int W) {
  constexpr int NL = PassGeom<T, L>::NL;
  ColTile ct;
  ct.CW = NL < W ? NL : W;
  ct.RPC = NL / ct.CW;
  ct.w = line % ct.CW;
  ct.rsub = line / ct.CW;
  return ct;
}

// ---- y forward: bufA[z][y < Ny][.] -> bufB[z][ky][.]
template <typename T, int L>
__global__ void __launch_bounds__(256) k_yfwd(HotDev h) {
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  T2 *tw, *xb;
  pass_prologue<T, L>(tw, xb, (const T2*)h.twy_tab, line);
  const int W = 8 * h.Nx, Ny = h.Ny;
  const ColTile ct = col_tile<T, L>(line, W);
  const int zi = blockIdx.y * ct.RPC + ct.rsub;
  const bool act = zi < h.nzocc;
  const int z = act ? h.zplanes[zi] : 0;
  const int b = blockIdx.z;
  const int64_t col = (int64_t)blockIdx.x * ct.CW + ct.w;
  const T2* __restrict__ in = (const T2*)h.bufA + b * h.sA + (int64_t)z * Ny * W + col;
  T2 v[G::E];
#pragma unroll
  for (int i = 0; i < G::E; ++i) {   // y < Ny = L/2  <=>  n2 < R2/2
    const int y = G::TL::in_index(t, i);
    v[i] = (act && i % G::R2 < G::R2 / 2) ? in[(int64_t)y * W] : mk<T2>(0, 0);
  }
  fwd_fft<T2, L>(v, xb, tw, t);
  if (!act) return;
  T2* __restrict__ out = (T2*)h.bufB + b * h.sB + (int64_t)z * L * W + col;
#pragma unroll
  for (int i = 0; i < G::E; ++i) out[(int64_t)TwoLevel<G::R2, G::R1>::in_index(t, i) * W] = v[i];
}

// ---- y inverse: bufB[z][ky][.] -> bufC[z][y < Ny, occupied][.]
template <typename T, int L>
__global__ void __launch_bounds__(256) k_yinv(HotDev h) {
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  T2 *tw, *xb;
  pass_prologue<T, L>(tw, xb, (const T2*)h.twy_tab, line);
  const int W = 8 * h.Nx, Ny = h.Ny;
  const ColTile ct = col_tile<T, L>(line, W);
  const int zi = blockIdx.y * ct.RPC + ct.rsub;
  const bool act = zi < h.nzocc;
  const int z = act ? h.zplanes[zi] : 0;
  const int b = blockIdx.z;
  const int64_t col = (int64_t)blockIdx.x * ct.CW + ct.w;
  const T2* __restrict__ in = (const T2*)h.bufB + b * h.sB + (int64_t)z * L * W + col;
  T2 v[G::E];
#pragma unroll
  for (int i = 0; i < G::E; ++i) v[i] = act ? in[(int64_t)G::TL::in_index(t, i) * W] : mk<T2>(0, 0);
  inv_fft<T2, L>(v, xb, tw, t);
  if (!act) return;
  T2* __restrict__ out = (T2*)h.bufC + b * h.sA + (int64_t)z * Ny * W + col;
  const uint8_t* occ = h.line_occ + (int64_t)z * Ny;
#pragma unroll
  for (int i = 0; i < G::E; ++i) {   // y < Ny  <=>  k1 < R1/2 in D(R2,R1)
    const int y = TwoLevel<G::R2, G::R1>::in_index(t, i);
    if (i % G::R1 < (G::R1 + 1) / 2 && y < Ny && occ[y]) out[(int64_t)y * W] = v[i];
  }
}

// ---- z forward * H_hat * z inverse, in place on bufB (occupied planes only)
template <typename T, int L, bool FULLZ>
__global__ void __launch_bounds__(256, (L <= 256 && sizeof(T) == 4) ? 3 : 1) k_zconv(HotDev h) {
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  __builtin_assume(t < G::T);
  const int W = 8 * h.Nx, Nx = h.Nx, Ny = h.Ny, Nz = h.Nz, Ny2 = 2 * h.Ny;
  const ColTile ct = col_tile<T, L>(line, W);
  const int b = blockIdx.z;
  // prefetch this CTA's spectrum slab [rsub][kz][kx - kx0] into shared memory
  // (cp.async, overlaps the column loads and the forward transform)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* hs = reinterpret_cast<T2*>(smem_raw) + L + (size_t)G::NL * G::XB;
  const int nkx = ct.CW / 4, kx0 = (blockIdx.x * ct.CW) / 4;
  {
    const T2* __restrict__ Hb = (const T2*)h.Hoct + b * h.sH;
    const int n = ct.RPC * L * nkx;
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const int r = idx / (L * nkx), kz = (idx / nkx) % L, kxl = idx % nkx;
      const int kyy = blockIdx.y * ct.RPC + r;
      const int kyf = kyy <= Ny ? kyy : Ny2 - kyy;
      const int kx = kx0 + kxl;
      const int kxf = kx <= Nx ? kx : 2 * Nx - kx;
      const int kzf = kz <= Nz ? kz : 2 * Nz - kz;
      if (kyy < Ny2) cp_async(hs + idx, Hb + ((int64_t)kyf * (Nz + 1) + kzf) * (Nx + 1) + kxf);
    }
  }
  T2 *tw, *xb;
  pass_prologue<T, L>(tw, xb, (const T2*)h.twz_tab, line);
  const int ky = blockIdx.y * ct.RPC + ct.rsub;
  const bool act = ky < Ny2;
  const int64_t col = (int64_t)blockIdx.x * ct.CW + ct.w;
  const int64_t zs = (int64_t)Ny2 * W;
  T2* __restrict__ g = (T2*)h.bufB + b * h.sB + (int64_t)(act ? ky : 0) * W + col;
  const uint8_t* __restrict__ zocc = h.zocc;
  // input distribution D(R1,R2): z = t + T a + R1 n2 < Nz = L/2  <=>  n2 < R2/2
  T2 v[G::E];
#pragma unroll
  for (int i = 0; i < G::E; ++i) {
    const int z = G::TL::in_index(t, i);
    if (i % G::R2 < G::R2 / 2) v[i] = (act && (FULLZ || zocc[z])) ? g[z * zs] : mk<T2>(0, 0);
    else v[i] = mk<T2>(0, 0);
  }
  fwd_fft<T2, L>(v, xb, tw, t);
  cp_async_wait_all();
  __syncthreads();
  {  // spectrum multiply (slab in shared memory, 1/M folded into H)
    const T2* hl = hs + (size_t)ct.rsub * L * nkx + (ct.w >> 2);
#pragma unroll
    for (int i = 0; i < G::E; ++i) {
      const int kz = TwoLevel<G::R2, G::R1>::in_index(t, i);
      v[i] = cmul(v[i], hl[kz * nkx]);
    }
  }
  inv_fft_swapped<T2, L>(v, xb, tw, t);
  if (!act) return;
#pragma unroll
  for (int i = 0; i < G::E; ++i) {
    const int z = G::TL::in_index(t, i);
    if (i % G::R2 < G::R2 / 2 && (FULLZ || zocc[z])) g[z * zs] = v[i];
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

// Single right-hand side: lanes stride the stencil nodes and the near row.
template <typename T>
__global__ void __launch_bounds__(256) k_interp_near1(HotDev h, const typename CT<T>::T2* __restrict__ x,
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
    const T4 w = ((const T4*)h.lam)[(int64_t)m * h.p3 + sl];
    const T2* ph = (const T2*)h.phi + lin * h.batch * 4;   // [node][channel][slot], slot 0
    const int pb = h.batch;
    const T2 p0 = ph[0], p1 = ph[pb], p2 = ph[2 * pb], p3 = ph[3 * pb];
    aA.x += w.x * p0.x + w.y * p1.x + w.z * p2.x;
    aA.y += w.x * p0.y + w.y * p1.y + w.z * p2.y;
    aR.x += w.w * p3.x;
    aR.y += w.w * p3.y;
  }
  const T2* __restrict__ cv = (const T2*)h.cval;
  const int kb = h.rowptr[m], ke = h.rowptr[m + 1];
#pragma unroll 4
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
      const R al = (R)cb.alpha_im[0], be = (R)cb.beta[0];
      const R ux = aA.x - be * aR.x, uy = aA.y - be * aR.y;
      y0[m] = mk<T2>(-al * uy, al * ux);   // (j alpha) * u
    } else {
      if (y0) y0[m] = aA;
      if (y1) y1[m] = mk<T2>(-aR.x, -aR.y);
    }
  }
}

// BB right-hand sides (batch-interleaved xt[n * BB + b], phi[(lin * slots + b)
// * 4 + c]): lane = (group g, columns b0..b0+V-1) with V complex per 16-byte
// load; the 32/(BB/V) groups stride the stencil nodes and the near row, the
// lanes of a group read one contiguous x row per near entry.
template <typename T2, int V> struct VecT;
template <> struct VecT<float2, 2> { using type = float4; };
template <> struct VecT<double2, 1> { using type = double2; };

template <typename T, int BB>
__global__ void __launch_bounds__(256) k_interp_near(HotDev h, const typename CT<T>::T2* __restrict__ xt,
                                                     typename CT<T>::T2* __restrict__ y0, Combine cb) {
  using T2 = typename CT<T>::T2;
  using T4 = typename CT<T>::T4;
  constexpr int V = sizeof(T2) == 8 ? 2 : 1;       // complex per 16-byte load
  constexpr int LG = BB / V;                         // lanes per group
  constexpr int NG = 32 / LG;                        // groups per warp
  using VT = typename VecT<T2, V>::type;
  const int lane = threadIdx.x & 31;
  const int b0 = (lane % LG) * V, g = lane / LG;
  const int m = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (m >= h.nb) return;
  T2 aA[V], aR[V];
#pragma unroll
  for (int v = 0; v < V; ++v) { aA[v] = mk<T2>(0, 0); aR[v] = mk<T2>(0, 0); }
  const int64_t ns = (int64_t)h.batch * 4;
  for (int sl = g; sl < h.p3; sl += NG) {
    const int p = h.p;
    const int i = sl % p, j = (sl / p) % p, k = sl / (p * p);
    const int64_t lin = (int64_t)h.rwg_base[m] + i + (int64_t)h.Nx * (j + (int64_t)h.Ny * k);
    const T4 w = ((const T4*)h.lam)[(int64_t)m * h.p3 + sl];
    // phi[node][channel][slot]: a group's lanes read one contiguous channel row
    const T2* phn = (const T2*)h.phi + lin * ns + b0;
    T2 pv[4 * V];   // pv[4 v + c] = channel c of column b0 + v
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const VT u = *(const VT*)(phn + (int64_t)c * h.batch);
      if constexpr (V == 2) {
        pv[c] = mk<T2>(u.x, u.y);
        pv[4 + c] = mk<T2>(u.z, u.w);
      } else {
        pv[c] = u;
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const T2 p0 = pv[4 * v], p1 = pv[4 * v + 1], p2 = pv[4 * v + 2], p3 = pv[4 * v + 3];
      aA[v].x += w.x * p0.x + w.y * p1.x + w.z * p2.x;
      aA[v].y += w.x * p0.y + w.y * p1.y + w.z * p2.y;
      aR[v].x += w.w * p3.x;
      aR[v].y += w.w * p3.y;
    }
  }
  // near row: the warp loads 32 entries (col, C) coalesced per chunk, then
  // each group takes every NG-th of them via shuffles, so the chunk's x-row
  // loads are independent and issue back to back.
  const T2* __restrict__ cv = (const T2*)h.cval;
  const int kb = h.rowptr[m], ke = h.rowptr[m + 1];
  for (int base = kb; base < ke; base += 32) {
    const int kk = base + lane;
    const bool ok = kk < ke;
    const int mycol = ok ? h.col[kk] : 0;
    const T2 myc = ok ? cv[kk] : mk<T2>(0, 0);
#pragma unroll
    for (int j = 0; j < 32; j += NG) {
      const int src = j + g;
      const int n = __shfl_sync(0xffffffffu, mycol, src);
      T2 c;
      c.x = __shfl_sync(0xffffffffu, myc.x, src);
      c.y = __shfl_sync(0xffffffffu, myc.y, src);
      // one load instruction per group: each touches a single 8*BB-byte row
      // (a multi-line load costs ~2 L1 cycles per line, a single-line one 1)
      VT u;
#pragma unroll
      for (int gg = 0; gg < NG; ++gg)
        if (g == gg) u = *(const VT*)(xt + (int64_t)n * BB + b0);   // entries past the row: c = 0
      T2 xv[V];
      if constexpr (V == 2) {
        xv[0] = mk<T2>(u.x, u.y);
        xv[1] = mk<T2>(u.z, u.w);
      } else {
        xv[0] = u;
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        aA[v].x += c.x * xv[v].x; aA[v].y += c.x * xv[v].y;
        aR[v].x += c.y * xv[v].x; aR[v].y += c.y * xv[v].y;
      }
    }
  }
#pragma unroll
  for (int o = LG; o < 32; o <<= 1) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      aA[v].x += __shfl_xor_sync(0xffffffffu, aA[v].x, o);
      aA[v].y += __shfl_xor_sync(0xffffffffu, aA[v].y, o);
      aR[v].x += __shfl_xor_sync(0xffffffffu, aR[v].x, o);
      aR[v].y += __shfl_xor_sync(0xffffffffu, aR[v].y, o);
    }
  }
  if (g == 0) {
    using R = decltype(T2::x);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int b = b0 + v;
      if (b < cb.B) {
        const R al = (R)cb.alpha_im[b], be = (R)cb.beta[b];
        const R ux = aA[v].x - be * aR[v].x, uy = aA[v].y - be * aR[v].y;
        y0[b * cb.ystride + m] = mk<T2>(-al * uy, al * ux);   // (j alpha) * u
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
  constexpr size_t sm = pass_smem<T, L>();
  constexpr int RPC = PassGeom<T, L>::NL / 4;
  dim3 g((unsigned)((h.nlines + RPC - 1) / RPC), (unsigned)B);
  if (!inv) {
    set_smem(k_xfwd<T, L>, sm);
    k_xfwd<T, L><<<g, PassGeom<T, L>::NT, sm, s>>>(h);
  } else {
    set_smem(k_xinv<T, L>, sm);
    k_xinv<T, L><<<g, PassGeom<T, L>::NT, sm, s>>>(h);
  }
  AIMX_CHECK_LAUNCH();
}

template <typename T, int L> dim3 col_grid(int W, int rows, int B) {
  constexpr int NL = PassGeom<T, L>::NL;
  const int CW = NL < W ? NL : W;
  const int RPC = NL / CW;
  return dim3((unsigned)(W / CW), (unsigned)((rows + RPC - 1) / RPC), (unsigned)B);
}

template <typename T, int L>
void run_y(const HotDev& h, bool inv, int B, cudaStream_t s) {
  constexpr size_t sm = pass_smem<T, L>();
  dim3 g = col_grid<T, L>(8 * h.Nx, h.nzocc, B);
  if (!inv) {
    set_smem(k_yfwd<T, L>, sm);
    k_yfwd<T, L><<<g, PassGeom<T, L>::NT, sm, s>>>(h);
  } else {
    set_smem(k_yinv<T, L>, sm);
    k_yinv<T, L><<<g, PassGeom<T, L>::NT, sm, s>>>(h);
  }
  AIMX_CHECK_LAUNCH();
}

template <typename T, int L>
void run_z(const HotDev& h, int B, cudaStream_t s) {
  // + spectrum slab: NL lines x L / 4 complex (RPC * L * CW / 4)
  constexpr size_t sm = pass_smem<T, L>() + sizeof(typename CT<T>::T2) * (size_t)PassGeom<T, L>::NL * L / 4;
  dim3 g = col_grid<T, L>(8 * h.Nx, 2 * h.Ny, B);
  if (h.nzocc == h.Nz) {
    set_smem(k_zconv<T, L, true>, sm);
    k_zconv<T, L, true><<<g, PassGeom<T, L>::NT, sm, s>>>(h);
  } else {
    set_smem(k_zconv<T, L, false>, sm);
    k_zconv<T, L, false><<<g, PassGeom<T, L>::NT, sm, s>>>(h);
  }
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

template <int BB> constexpr int bucket_ok() { return BB; }
inline int batch_bucket(int B) { return B <= 1 ? 1 : (B <= 2 ? 2 : (B <= 4 ? 4 : (B <= 8 ? 8 : 16))); }

template <typename T>
void run_interleave(const HotDev& h, const void* x, const Combine& c, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const int BB = batch_bucket(c.B);
  const int64_t n = (int64_t)h.nb * BB;
  k_interleave<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h.nb, c.B, BB, (const T2*)x, c.xstride,
                                                              (T2*)h.xt);
  AIMX_CHECK_LAUNCH();
}

template <typename T>
void run_gather_b(const HotDev& h, int B, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const unsigned g = (unsigned)(((int64_t)h.nocc * 32 + 255) / 256);
  const T2* xt = (const T2*)h.xt;
  switch (batch_bucket(B)) {
    case 2: k_gather_b<T, 2><<<g, 256, 0, s>>>(h, xt, B); break;
    case 4: k_gather_b<T, 4><<<g, 256, 0, s>>>(h, xt, B); break;
    case 8: k_gather_b<T, 8><<<g, 256, 0, s>>>(h, xt, B); break;
    default: k_gather_b<T, 16><<<g, 256, 0, s>>>(h, xt, B); break;
  }
  AIMX_CHECK_LAUNCH();
}

template <typename T>
void run_interp(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const unsigned g = (unsigned)(((int64_t)h.nb * 32 + 255) / 256);
  if (c.B == 1) {
    k_interp_near1<T><<<g, 256, 0, s>>>(h, (const T2*)x, (T2*)y0, (T2*)y1, c);
    AIMX_CHECK_LAUNCH();
    return;
  }
  if (c.mode != 0) throw Error(AIMX_E_INTERNAL, "batched parts not supported");
  const T2* xt = (const T2*)h.xt;   // interleaved by run_interleave earlier in the matvec
  switch (batch_bucket(c.B)) {
    case 2: k_interp_near<T, 2><<<g, 256, 0, s>>>(h, xt, (T2*)y0, c); break;
    case 4: k_interp_near<T, 4><<<g, 256, 0, s>>>(h, xt, (T2*)y0, c); break;
    case 8: k_interp_near<T, 8><<<g, 256, 0, s>>>(h, xt, (T2*)y0, c); break;
    default: k_interp_near<T, 16><<<g, 256, 0, s>>>(h, xt, (T2*)y0, c); break;
  }
  AIMX_CHECK_LAUNCH();
}

template <typename T>
void hot_matvec(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s,
                Profiler* prof) {
  if (c.B < 1 || c.B > h.batch || c.B > kMaxBatch) throw Error(AIMX_E_INTERNAL, "bad batch");
  const int Lx = 2 * h.Nx, Ly = 2 * h.Ny, Lz = 2 * h.Nz, B = c.B;
  {
    StageScope sc(prof, 1, s);
    if (B == 1) {
      run_gather<T>(h, x, c.xstride, B, s);
    } else {
      run_interleave<T>(h, x, c, s);
      run_gather_b<T>(h, B, s);
    }
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
