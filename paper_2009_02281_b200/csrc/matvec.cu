// The AIMx hot path on the B200 (S2-S5), batched over B frequency points:
//
//   k_interleave  the B right-hand sides batch-interleaved: xt[n][b]
//   k_gather(_b)  S2: projection P x as a gather over the transposed
//                 (node-major) stencil CSR -- a warp or lane group per occupied
//                 grid node, fixed-order shuffle reduction, no atomics -- into
//                 dense occupied x-lines S[line][x][4]
//   k_xfwd        zero-padded forward FFT along x of the occupied lines
//   k_yzconv      (short y and z) y fwd, z fwd * H_hat * z inv, y inv in one
//                 kernel over shared-memory column tiles; otherwise:
//   k_yfwd        forward FFT along y (input rows y < N_y, zero padded)
//   k_zconv(_tma) forward FFT along z, times the spectrum H_hat (octant,
//                 already scaled by 1/M), inverse FFT along z, cropped to
//                 z < N_z (TMA tensor copies when every z plane is occupied)
//   k_yinv        inverse FFT along y, cropped to y < N_y (occupied lines only)
//   k_xinv        inverse FFT along x, cropped to x < N_x -> potentials phi
//   k_interp_near S4 + S5 on row groups (NearGroups): interpolation W = P^T of
//                 the 4 potentials and the near correction C = L_s,NR - L_s,P,
//                 coefficient stream by TMA bulk copies, then the EFIE combine
//                 y = -j w mu0 (y^A - k0^-2 y^rho).
// Every kernel is launched with programmatic dependent launch (fft.cuh).
// The slab-decomposed variant (slab_matvec) runs the same kernels per rank.
//
// P:198-200 (W H P, "accelerated with FFTs", applied on the entire grid);
// eq:LAIMx P:283; eq:EFIEAIMx P:288.  Grid data are complex, 4 channels
// (x, y, z, rho) innermost: element ((z * Ny' + y) * Nx' + x) * 4 + c.
// Pruning (exact, reading R12): lines/planes with no occupied node are never
// transformed; their data are identically zero and are never read as input.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "aimx_internal.h"
#include "fft.cuh"
#include "fft_reg.cuh"
#include "tma.cuh"

namespace aimx {

namespace {

// ------------------------------------------------------------------ S2 gather
template <typename T, int G>
__global__ void __launch_bounds__(256) k_gather(HotDev h, const typename CT<T>::T2* __restrict__ x,
                                                int64_t xstride) {
  pdl_wait();
  pdl_trigger();
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
  if (act && gl == 0) {   // nc = 3: the channels (x, y, rho) of a planar grid
    T2* dst = (T2*)h.S + b * h.sS + ((int64_t)h.node_line[q] * h.Nx + h.node_lin[q] % h.Nx) * h.nc;
    dst[0] = a0; dst[1] = a1;
    if (h.nc == 4) { dst[2] = a2; dst[3] = a3; }
    else dst[2] = a3;
  }
}

// S2 for BB right-hand sides at once (batch-interleaved xt[n * BB + b]):
// warp per occupied node, groups of BB/V lanes stride its entries (each entry's
// weights and RWG index read once for all columns), lanes cover columns.  The
// entries come in coalesced chunks of 32 (the next chunk's loaded while this
// one is used); within a chunk each group issues its x-row loads 8 at a time
// before the arithmetic (packed FFMA2 in fp32).
template <typename T, int BB>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 3 : 2) k_gather_b(HotDev h, const typename CT<T>::T2* __restrict__ xt,
                                                     int B) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using T4 = typename CT<T>::T4;
  constexpr int V = sizeof(T2) == 8 ? 2 : 1;
  constexpr int LG = BB / V, NG = 32 / LG;
  constexpr int PER = 32 / NG;             // entries of a chunk per group
  // loads in flight per batch: 4 (3 CTAs of 256 threads per SM; with 8 the
  // registers allowed 2 and the gather was latency bound at 22% occupancy)
  constexpr int QB = PER < 4 ? PER : 4;
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
  int myr = 0;
  T4 myw{0, 0, 0, 0};
  if (e0 + lane < e1) {
    myr = h.ent_rwg[e0 + lane];
    myw = ew[e0 + lane];
  }
  for (int base = e0; base < e1; base += 32) {
    const int nx = base + 32 + lane;
    const int cnt = e1 - base;   // entries left (the last chunk may be partial)
    int nr = 0;
    T4 nw{0, 0, 0, 0};
    if (nx < e1) {   // next chunk, in flight during this one
      nr = h.ent_rwg[nx];
      nw = ew[nx];
    }
#pragma unroll
    for (int jb = 0; jb < PER; jb += QB) {
      if (jb * NG >= cnt) break;   // warp-uniform: no entry of this batch exists
      VT u[QB];
      T4 w[QB];
#pragma unroll
      for (int qq = 0; qq < QB; ++qq) {
        const int src = (jb + qq) * NG + g;   // entries past the node carry zero weights
        w[qq].x = __shfl_sync(0xffffffffu, myw.x, src);
        w[qq].y = __shfl_sync(0xffffffffu, myw.y, src);
        w[qq].z = __shfl_sync(0xffffffffu, myw.z, src);
        w[qq].w = __shfl_sync(0xffffffffu, myw.w, src);
        const int rr = __shfl_sync(0xffffffffu, myr, src);
        u[qq] = *(const VT*)(xt + (int64_t)rr * BB + b0);
      }
#pragma unroll
      for (int qq = 0; qq < QB; ++qq) {
        T2 xv[V];
        if constexpr (V == 2) {
          xv[0] = mk<T2>(u[qq].x, u[qq].y);
          xv[1] = mk<T2>(u[qq].z, u[qq].w);
        } else {
          xv[0] = u[qq];
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
          axpy(a[v][0], w[qq].x, xv[v]);
          axpy(a[v][1], w[qq].y, xv[v]);
          axpy(a[v][2], w[qq].z, xv[v]);
          axpy(a[v][3], w[qq].w, xv[v]);
        }
      }
    }
    myr = nr;
    myw = nw;
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
    const int nc = h.nc;
    const int64_t off = ((int64_t)h.node_line[q] * h.Nx + h.node_lin[q] % h.Nx) * nc;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int b = b0 + v;
      if (b < B) {
        T2* dst = (T2*)h.S + b * h.sS + off;
        dst[0] = a[v][0]; dst[1] = a[v][1];
        if (nc == 4) { dst[2] = a[v][2]; dst[3] = a[v][3]; }
        else dst[2] = a[v][3];
      }
    }
  }
}

// ------------------------------------------------------------------ FFT passes
// Register-resident two-level FFTs (fft_reg.cuh).  Threads are mapped
// line-fastest (line = tid % NL, t = tid / NL) so that a warp's loads and
// stores cover consecutive grid columns; the per-line exchange uses one block
// barrier per transform.
template <typename S, int L, bool SMALL = false> struct PassGeom {
  static constexpr int R1 = Fac<L>::R1, R2 = Fac<L>::R2;
  using TL = TwoLevel<R1, R2>;
  static constexpr int T = TL::T, E = TL::E;
  // per-line exchange stride: bank-spread so that the lines and threads of a
  // half-warp (one shared-memory wavefront of 8-byte accesses: 16 lanes) hit
  // distinct 8-byte slots: a half-warp holds NL lines x 16/NL threads, so the
  // stride is 16/NL mod 16 -- 1 for 16 lines (T = 16), 2 for 8 lines (T = 32,
  // 256 threads), 4 for 4 lines (T = 32, SMALL: 128 threads).  (4 for 8 lines
  // put lines l and l + 4 on one slot: ncu counted 12.6 M excess store and
  // 13 M excess load wavefronts in the cfg5 planar y pass, 30% of its stalls.)
  static constexpr int XB = R1 > 1 ? ((TL::XB + 15) / 16) * 16 + (T == 32 ? (SMALL ? 4 : 2) : 1) : 0;
  static constexpr size_t BYTES256 = sizeof(typename CT<S>::T2) * (size_t)(256 / T) * XB;
  // threads per CTA; SMALL: one x row (4 channel lines) per CTA when rows are few
  static constexpr int NT = SMALL ? (4 * T > 64 ? 4 * T : 64) : (BYTES256 > 200 * 1024 ? 128 : 256);
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

// ASYNC: the twiddle table goes global -> shared by cp.async (one commit
// group) so its latency overlaps the pass's input loads; the kernel calls
// pass_ready() after issuing them, before the first transform.
template <typename T, int L, bool SMALL = false, bool ASYNC = false>
__device__ __forceinline__ void pass_prologue(typename CT<T>::T2*& tw, typename CT<T>::T2*& xb,
                                              const typename CT<T>::T2* __restrict__ gtw, int line) {
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L, SMALL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  tw = reinterpret_cast<T2*>(smem_raw);
  xb = tw + L + line * G::XB;
  if constexpr (ASYNC) {
    for (int i = threadIdx.x; i < L; i += blockDim.x) cp_async(tw + i, gtw + i);
    asm volatile("cp.async.commit_group;\n" ::);
  } else {
    for (int i = threadIdx.x; i < L; i += blockDim.x) tw[i] = gtw[i];
    __syncthreads();
  }
}
// every cp.async of this thread landed, and every thread's (block barrier)
__device__ __forceinline__ void pass_ready() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
}

template <typename T, int L, bool SMALL = false> constexpr size_t pass_smem() {
  using G = PassGeom<T, L, SMALL>;
  return sizeof(typename CT<T>::T2) * (L + (size_t)G::NL * G::XB);
}

// ---- x forward: occupied lines of S (x < Nx, zero padded) -> bufA[line_id][kx][c]
template <typename T, int L, bool SMALL>
__global__ void __launch_bounds__(256, (sizeof(T) == 4 && !SMALL) ? 3 : 1) k_xfwd(HotDev h) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L, SMALL>;
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  T2 *tw, *xb;
  pass_prologue<T, L, SMALL, true>(tw, xb, (const T2*)h.twx, line);
  const int b = blockIdx.y, nc = h.nc;   // lines = (grid line r, channel c < nc), c fastest
  const int gline = blockIdx.x * G::NL + line, r = gline / nc, c = gline - r * nc;
  const bool act = r < h.nlines;
  const int Nx = h.Nx;
  const T2* __restrict__ in = (const T2*)h.S + b * h.sS + (int64_t)(act ? r : 0) * Nx * nc + c;
  T2 v[G::E];
#pragma unroll
  for (int i = 0; i < G::E; ++i) {   // x < Nx = L/2  <=>  n2 < R2/2
    const int x = G::TL::in_index(t, i);
    v[i] = (act && i % G::R2 < G::R2 / 2) ? in[x * nc] : mk<T2>(0, 0);
  }
  pass_ready();
  fwd_fft<T2, L>(v, xb, tw, t);
  if (!act) return;
  T2* __restrict__ out = (T2*)h.bufA + b * h.sA + (int64_t)h.line_id[r] * L * nc + c;
#pragma unroll
  for (int i = 0; i < G::E; ++i) out[TwoLevel<G::R2, G::R1>::in_index(t, i) * nc] = v[i];
}

// ---- x inverse: bufC[line_id][kx][c] -> phi[line][x < Nx][c]
template <typename T, int L, bool SMALL>
__global__ void __launch_bounds__(256, (sizeof(T) == 4 && !SMALL) ? 3 : 1) k_xinv(HotDev h) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L, SMALL>;
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  T2 *tw, *xb;
  pass_prologue<T, L, SMALL, true>(tw, xb, (const T2*)h.twx, line);
  const int b = blockIdx.y, nc = h.nc;
  const int gline = blockIdx.x * G::NL + line, r = gline / nc, c = gline - r * nc;
  const bool act = r < h.nlines;
  const int lid = act ? h.line_id[r] : 0;
  const T2* __restrict__ in = (const T2*)h.bufC + b * h.sA + (int64_t)lid * L * nc + c;
  T2 v[G::E];
#pragma unroll
  for (int i = 0; i < G::E; ++i) v[i] = act ? in[G::TL::in_index(t, i) * nc] : mk<T2>(0, 0);
  pass_ready();
  inv_fft<T2, L>(v, xb, tw, t);
  if (!act) return;
  const int Nx = h.Nx;
  // phi layout [node][channel][slot] (slots = batch, complex)
  const int64_t ns = (int64_t)h.batch * nc;   // node stride
  const int plid = h.phi_line ? (act ? h.phi_line[r] : 0) : lid;   // line of phi (global grid)
  T2* __restrict__ out = (T2*)h.phi + (int64_t)c * h.batch + b + (int64_t)plid * Nx * ns;
#pragma unroll
  for (int i = 0; i < G::E; ++i) {   // x < Nx  <=>  k1 < R1/2 in D(R2,R1)
    const int x = TwoLevel<G::R2, G::R1>::in_index(t, i);
    if (i % G::R1 < (G::R1 + 1) / 2 && x < Nx) out[x * ns] = v[i];
  }
}

// ---- x inverse, batched (B >= 4): the CTA's lines are the NCH channels x 4
// consecutive slots of one grid line, so both sides move whole 32-byte
// sectors: each read or write of the grid rows covers the channels of a
// slot's point ([slot][line][x][c]), each write of phi 4 consecutive slots of
// a channel ([node][c][slot]).  With the per-slot mapping of k_xinv every phi
// write was a lone 8-byte piece of a sector (cfg5, 32 columns: 766 us, issue
// 7%).  NCH = the stored channels: 4, or 3 on a planar grid (h.nc).
template <typename T, int L, int NCH = 4> struct XinvB {
  static constexpr int T_ = TwoLevel<Fac<L>::R1, Fac<L>::R2>::T;
  static constexpr int NL = 4 * NCH, NT = NL * T_;
  static constexpr int XB = PassGeom<T, L>::XB;   // (3 mod 16 for the 12-line CTA measured 199 -> 207 us on cfg5)
  static constexpr size_t SMEM = sizeof(typename CT<T>::T2) * (L + (size_t)NL * XB);
};
template <typename T, int L, int NCH>
__global__ void __launch_bounds__(XinvB<T, L, NCH>::NT, (sizeof(T) == 4 && NCH == 3) ? 2 : 1) k_xinv_b(HotDev h, int B) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  using X = XinvB<T, L, NCH>;
  const int line = threadIdx.x % X::NL, t = threadIdx.x / X::NL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* xb = tw + L + line * X::XB;
  for (int i = threadIdx.x; i < L; i += X::NT) cp_async(tw + i, (const T2*)h.twx + i);   // lands behind the input loads
  const int r = blockIdx.x, c = line % NCH, b = blockIdx.y * 4 + line / NCH;
  const bool act = b < B;
  const int lid = h.line_id[r];
  const T2* __restrict__ in = (const T2*)h.bufC + (int64_t)(act ? b : 0) * h.sA + (int64_t)lid * L * NCH + c;
  T2 v[G::E];
#pragma unroll
  for (int i = 0; i < G::E; ++i) v[i] = act ? in[G::TL::in_index(t, i) * NCH] : mk<T2>(0, 0);
  pass_ready();
  inv_fft<T2, L>(v, xb, tw, t);
  if (!act) return;
  const int Nx = h.Nx;
  const int64_t ns = (int64_t)h.batch * NCH;   // phi node stride (complex): [node][channel][slot]
  const int plid = h.phi_line ? h.phi_line[r] : lid;
  T2* __restrict__ out = (T2*)h.phi + (int64_t)c * h.batch + b + (int64_t)plid * Nx * ns;
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
// column tile width: the largest power of two <= NL that divides W (W = 8 N_x,
// or 4 x the kx slab: a multiple of 8; radix-3 grids such as N_x = 24 give W
// = 192, not a multiple of the 128 lines of a length-48 pass)
__host__ __device__ __forceinline__ int col_width(int W, int NL) {
  int cw = NL < W ? NL : W;
  while (cw > 8 && W % cw) cw >>= 1;
  return cw;
}
template <typename T, int L> __device__ __forceinline__ ColTile col_tile(int line, int W) {
  constexpr int NL = PassGeom<T, L>::NL;
  ColTile ct;
  ct.CW = col_width(W, NL);
  ct.RPC = NL / ct.CW;
  ct.w = line % ct.CW;
  ct.rsub = line / ct.CW;
  return ct;
}

// ---- y forward: bufA[z][y < Ny][.] -> bufB[z][ky][.]
template <typename T, int L>
__global__ void __launch_bounds__(256) k_yfwd(HotDev h) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  T2 *tw, *xb;
  pass_prologue<T, L, false, true>(tw, xb, (const T2*)h.twy_tab, line);
  const int W = h.W, Ny = h.Ny;
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
  pass_ready();
  fwd_fft<T2, L>(v, xb, tw, t);
  if (!act) return;
  T2* __restrict__ out = (T2*)h.bufB + b * h.sB + (int64_t)z * L * W + col;
#pragma unroll
  for (int i = 0; i < G::E; ++i) out[(int64_t)TwoLevel<G::R2, G::R1>::in_index(t, i) * W] = v[i];
}

// ---- y inverse: bufB[z][ky][.] -> bufC[z][y < Ny, occupied][.]
template <typename T, int L>
__global__ void __launch_bounds__(256) k_yinv(HotDev h) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  T2 *tw, *xb;
  pass_prologue<T, L, false, true>(tw, xb, (const T2*)h.twy_tab, line);
  const int W = h.W, Ny = h.Ny;
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
  pass_ready();
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
// Each CTA walks ZROWS consecutive row sets (of RPC ky rows each) of its
// column tile, so the twiddle table and the per-thread spectrum-slab offsets
// are set up once; the slab of the next row set is prefetched with cp.async
// while the current one is transformed.
constexpr int ZROWS = 8;
template <typename T, int L, bool FULLZ>
__global__ void __launch_bounds__(256, (L <= 256 && sizeof(T) == 4) ? 3 : 1) k_zconv(HotDev h) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  constexpr int NPF = G::E / 4;   // slab elements per thread: (RPC L CW/4) / NT
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  __builtin_assume(t < G::T);
  const int W = h.W, Nx = h.Nx, Ny = h.Ny, Nz = h.Nz, Ny2 = 2 * h.Ny;
  const ColTile ct = col_tile<T, L>(line, W);
  const int b = blockIdx.z;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* hs = reinterpret_cast<T2*>(smem_raw) + L + (size_t)G::NL * G::XB;   // [2][RPC][kz][kx - kx0]
  const int nkx = ct.CW / 4, kx0 = h.kx0 + (blockIdx.x * ct.CW) / 4;   // kx0: column slab offset
  const int nslab = ct.RPC * L * nkx;
  const T2* __restrict__ Hb = (const T2*)h.Hoct + b * h.sH;
  const int64_t kystride = (int64_t)(Nz + 1) * (Nx + 1);
  // this thread's slab elements: row-set-independent offset and row
  int64_t poff[NPF];
  int prow[NPF];
  {
    const int lgk = __ffs(nkx) - 1;   // nkx: power of two
#pragma unroll
    for (int k = 0; k < NPF; ++k) {
      const int idx = threadIdx.x + k * G::NT;
      const int kxl = idx & (nkx - 1), rest = idx >> lgk;
      const int kz = rest % L;   // L: compile-time power of two
      const int kx = kx0 + kxl;
      const int kxf = kx <= Nx ? kx : 2 * Nx - kx;
      const int kzf = kz <= Nz ? kz : 2 * Nz - kz;
      poff[k] = (int64_t)kzf * (Nx + 1) + kxf;
      prow[k] = rest / L;
    }
  }
  auto prefetch = [&](int rs, int buf) {
#pragma unroll
    for (int k = 0; k < NPF; ++k) {
      const int idx = threadIdx.x + k * G::NT;
      const int kyy = rs * ct.RPC + prow[k];
      const int kyf = kyy <= Ny ? kyy : Ny2 - kyy;
      if (idx < nslab && kyy < Ny2) cp_async(hs + buf * nslab + idx, Hb + (int64_t)kyf * kystride + poff[k]);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  T2 *tw, *xb;
  pass_prologue<T, L>(tw, xb, (const T2*)h.twz_tab, line);
  const int64_t col = (int64_t)blockIdx.x * ct.CW + ct.w;
  const int64_t zs = (int64_t)Ny2 * W;
  const uint8_t* __restrict__ zocc = h.zocc;
  const int rs0 = blockIdx.y * ZROWS;
  prefetch(rs0, 0);
  for (int it = 0; it < ZROWS; ++it) {
    const int rs = rs0 + it;
    if (rs * ct.RPC >= Ny2) break;   // uniform over the CTA
    if (it + 1 < ZROWS && (rs + 1) * ct.RPC < Ny2) prefetch(rs + 1, (it + 1) & 1);
    const int ky = rs * ct.RPC + ct.rsub;
    const bool act = ky < Ny2;
    T2* __restrict__ g = (T2*)h.bufB + b * h.sB + (int64_t)(act ? ky : 0) * W + col;
    // input distribution D(R1,R2): z = t + T a + R1 n2 < Nz = L/2  <=>  n2 < R2/2
    T2 v[G::E];
#pragma unroll
    for (int i = 0; i < G::E; ++i) {
      const int z = G::TL::in_index(t, i);
      if (i % G::R2 < G::R2 / 2) v[i] = (act && (FULLZ || zocc[z])) ? g[z * zs] : mk<T2>(0, 0);
      else v[i] = mk<T2>(0, 0);
    }
    fwd_fft<T2, L>(v, xb, tw, t);
    // this row set's slab has landed (the next one may still be in flight)
    if (it + 1 < ZROWS && (rs + 1) * ct.RPC < Ny2) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    {  // spectrum multiply (slab in shared memory, 1/M folded into H)
      const T2* hl = hs + (it & 1) * nslab + (size_t)ct.rsub * L * nkx + (ct.w >> 2);
#pragma unroll
      for (int i = 0; i < G::E; ++i) {
        const int kz = TwoLevel<G::R2, G::R1>::in_index(t, i);
        v[i] = cmul(v[i], hl[kz * nkx]);
      }
    }
    inv_fft_swapped<T2, L>(v, xb, tw, t);
    if (act) {
#pragma unroll
      for (int i = 0; i < G::E; ++i) {
        const int z = G::TL::in_index(t, i);
        if (i % G::R2 < G::R2 / 2 && (FULLZ || zocc[z])) g[z * zs] = v[i];
      }
    }
    __syncthreads();   // slab buffer (it & 1) is refilled two row sets later; xb reuse
  }
}

// ---- z conv with TMA (all z planes occupied, N_z <= 256, one ky row per
// CTA step): per row set ONE tensor copy brings the CTA's [z < N_z][16 columns]
// block into shared memory (mbarrier), double-buffered one row set ahead; the
// results go back with one tensor store from the same buffer.  Loads and
// stores never occupy registers, so the transforms of one row set overlap the
// HBM traffic of the next.
// z-pass geometry of the TMA kernel: 16 lines (columns) per CTA in fp32, 8 in
// fp64 (smaller CTAs, more of them resident)
template <typename S, int L> struct ZGeom {
  static constexpr int R1 = Fac<L>::R1, R2 = Fac<L>::R2;
  using TL = TwoLevel<R1, R2>;
  static constexpr int T = TL::T, E = TL::E;
  static constexpr int XB = PassGeom<S, L>::XB;
  static constexpr int NL = sizeof(S) == 4 ? 16 : 8, NT = NL * T;   // (measured on cfg3)
};
// CURL (the double-layer operator's grid part, eq:KAIMx): three spectra (the
// gradient components d_a G), a [kz][column] exchange of the channels
template <typename T, int L, bool CURL = false> struct ZTma {
  using G = ZGeom<T, L>;
  static constexpr int CW = G::NL;   // columns per CTA (one ky row per step)
  static constexpr int NS = CURL ? 3 : 1;   // spectra
  static constexpr size_t XCH = CURL ? sizeof(typename CT<T>::T2) * (size_t)L * CW : 0;   // channel exchange
  static constexpr size_t OFF_HS = sizeof(typename CT<T>::T2) * (L + (size_t)G::NL * G::XB) + XCH;
  static constexpr int KZ = L / 2 + 1;   // stored kz (the octant; kz > L/2 mirrors on read)
  static constexpr int NPF = (KZ * (CW / 4) + G::NT - 1) / G::NT;   // slab elements per thread and spectrum
  static constexpr size_t HSB = sizeof(typename CT<T>::T2) * (size_t)NS * KZ * CW / 4;   // one slab
  static constexpr size_t OFF_IN = (OFF_HS + 2 * HSB + 127) / 128 * 128;   // TMA: 128-byte aligned
  __host__ __device__ static size_t inb(int Nz) { return sizeof(typename CT<T>::T2) * (size_t)Nz * CW; }
  // input ring depth: 3 (two row sets in flight) when two CTAs still fit an SM
  __host__ __device__ static int nbuf(int Nz) { return OFF_IN + 3 * inb(Nz) + 24 + 128 <= 112 * 1024 ? 3 : 2; }
  __host__ __device__ static size_t smem(int Nz) { return OFF_IN + nbuf(Nz) * inb(Nz) + 24 + 128; }
};

template <typename T, int L, bool CURL = false>
__global__ void __launch_bounds__(ZGeom<T, L>::NT, sizeof(T) == 4 ? 2 : 2) k_zconv_tma(HotDev h, const __grid_constant__ CUtensorMap tm) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using G = ZGeom<T, L>;
  using Z = ZTma<T, L, CURL>;
  constexpr int NPF = Z::NPF, CW = Z::CW, C0S = sizeof(T2) / 8;   // tensor elements per complex
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  __builtin_assume(t < G::T);
  const int Nx = h.Nx, Ny = h.Ny, Nz = h.Nz, Ny2 = 2 * h.Ny;
  const int b = blockIdx.z;
  extern __shared__ __align__(128) unsigned char smem_dyn[];
  // 128-byte aligned base by pointer arithmetic on the shared array (an
  // integer round trip would lose the address space: generic LD/ST for every
  // exchange and slab access, measured as 42% of the stall samples)
  unsigned char* smem_raw = smem_dyn + ((128u - (smem_u32(smem_dyn) & 127u)) & 127u);
  T2* hs = reinterpret_cast<T2*>(smem_raw + Z::OFF_HS);                        // [2][NS][kz <= Nz][kx - kx0]
  const int NB = Z::nbuf(Nz);
  T2* inb = reinterpret_cast<T2*>(smem_raw + Z::OFF_IN);                       // [NB][z][CW]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + Z::OFF_IN + NB * Z::inb(Nz));
  constexpr int nkx = CW / 4;
  const int kx0 = h.kx0 + (blockIdx.x * CW) / 4;
  constexpr int nslab1 = Z::KZ * nkx;   // one spectrum's slab: kz = 0..Nz (Nz = L/2 here)
  constexpr int nslab = Z::NS * nslab1;
  const T2* __restrict__ Hb = (const T2*)h.Hoct + b * h.sH;
  const int64_t noct = (int64_t)(Nx + 1) * (Ny + 1) * (Nz + 1);   // spectrum stride (CURL: d_x, d_y, d_z G)
  const int64_t kystride = (int64_t)(Nz + 1) * (Nx + 1);
  int64_t poff[NPF];
  {
    constexpr int LGK = CW == 64 ? 4 : (CW == 32 ? 3 : (CW == 16 ? 2 : (CW == 8 ? 1 : 0)));
#pragma unroll
    for (int k = 0; k < NPF; ++k) {
      const int idx = threadIdx.x + k * G::NT;
      const int kxl = idx & (nkx - 1), kz = min(idx >> LGK, Nz);
      const int kx = kx0 + kxl;
      const int kxf = kx <= Nx ? kx : 2 * Nx - kx;
      poff[k] = (int64_t)kz * (Nx + 1) + kxf;
    }
  }
  auto prefetch = [&](int ky, int buf) {
    const int kyf = ky <= Ny ? ky : Ny2 - ky;
#pragma unroll
    for (int a = 0; a < Z::NS; ++a)
#pragma unroll
      for (int k = 0; k < NPF; ++k) {
        const int idx = threadIdx.x + k * G::NT;
        if (idx < nslab1)
          cp_async(hs + buf * nslab + a * nslab1 + idx, Hb + a * noct + (int64_t)kyf * kystride + poff[k]);
      }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  const int col0 = blockIdx.x * CW, rs0 = blockIdx.y * ZROWS;
  const int nrs = min(ZROWS, Ny2 - rs0);
  const uint32_t bytes = (uint32_t)Z::inb(Nz);
  if (threadIdx.x == 0) {
    for (int k = 0; k < NB; ++k) mbar_init(bar + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* xb = tw + L + line * G::XB;
  for (int i = threadIdx.x; i < L; i += G::NT) tw[i] = ((const T2*)h.twz_tab)[i];
  __syncthreads();
  if (threadIdx.x == 0)   // rows rs0 .. rs0 + NB - 2 in flight before the loop
    for (int k = 0; k < NB - 1 && k < nrs; ++k) {
      mbar_arrive_expect_tx(bar + k, bytes);
      tma_load4(inb + (size_t)k * Nz * CW, &tm, col0 * C0S, rs0 + k, 0, b, bar + k);
    }
  prefetch(rs0, 0);
  for (int it = 0; it < nrs; ++it) {
    const int ky = rs0 + it, buf = it & 1, ring = it % NB;
    T2* ib = inb + (size_t)ring * Nz * CW;
    if (it + 1 < nrs) prefetch(ky + 1, buf ^ 1);
    if (threadIdx.x == 0 && it + NB - 1 < nrs) {
      const int nr = (it + NB - 1) % NB;   // = the ring slot of row set it-1
      bulk_wait_read0();                   // whose store has read it
      mbar_arrive_expect_tx(bar + nr, bytes);
      tma_load4(inb + (size_t)nr * Nz * CW, &tm, col0 * C0S, ky + NB - 1, 0, b, bar + nr);
    }
    mbar_wait(bar + ring, (uint32_t)(it / NB) & 1u);
    // input distribution D(R1,R2): z = t + T a + R1 n2 < Nz = L/2  <=>  n2 < R2/2
    T2 v[G::E];
#pragma unroll
    for (int i = 0; i < G::E; ++i) {
      const int z = G::TL::in_index(t, i);
      v[i] = (i % G::R2 < G::R2 / 2) ? ib[z * CW + line] : mk<T2>(0, 0);
    }
    fwd_fft<T2, L>(v, xb, tw, t);
    if constexpr (CURL) {   // this thread's z spectrum of its column, to the channel exchange
      T2* xs = reinterpret_cast<T2*>(smem_raw + Z::OFF_HS - Z::XCH);   // [kz][column]
#pragma unroll
      for (int i = 0; i < G::E; ++i) xs[TwoLevel<G::R2, G::R1>::in_index(t, i) * CW + line] = v[i];
    }
    if (it + 1 < nrs) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    if constexpr (CURL) {
      // Phi_c = (G_hat x J_hat)_c = sum_ab eps_cab G_hat_a J_hat_b at this (kx, ky, kz);
      // G_hat_a is odd along a: its octant value changes sign past N_a
      const T2* xs = reinterpret_cast<const T2*>(smem_raw + Z::OFF_HS - Z::XCH);
      const int c = line & 3, c0 = line & ~3;
      const int kx = kx0 + (line >> 2);
      const T sx = kx > Nx ? T(-1) : T(1), sy = ky > Ny ? T(-1) : T(1);
      const T2* hl = hs + buf * nslab + (line >> 2);
#pragma unroll
      for (int i = 0; i < G::E; ++i) {
        const int kz = TwoLevel<G::R2, G::R1>::in_index(t, i);
        const int kzf = kz <= L / 2 ? kz : L - kz;
        const T sz = kz > L / 2 ? T(-1) : T(1);
        const T2 jx = xs[kz * CW + c0], jy = xs[kz * CW + c0 + 1], jz = xs[kz * CW + c0 + 2];
        const T2 gx0 = hl[kzf * nkx], gy0 = hl[nslab1 + kzf * nkx], gz0 = hl[2 * nslab1 + kzf * nkx];
        const T2 gx = mk<T2>(sx * gx0.x, sx * gx0.y), gy = mk<T2>(sy * gy0.x, sy * gy0.y),
                 gz = mk<T2>(sz * gz0.x, sz * gz0.y);
        if (c == 0) v[i] = csub(cmul(gy, jz), cmul(gz, jy));
        else if (c == 1) v[i] = csub(cmul(gz, jx), cmul(gx, jz));
        else if (c == 2) v[i] = csub(cmul(gx, jy), cmul(gy, jx));
        else v[i] = mk<T2>(0, 0);
      }
    } else {  // spectrum multiply (slab in shared memory, 1/M folded into H)
      const T2* hl = hs + buf * nslab + (line >> 2);
#pragma unroll
      for (int i = 0; i < G::E; ++i) {
        const int kz = TwoLevel<G::R2, G::R1>::in_index(t, i);
        v[i] = cmul(v[i], hl[(kz <= L / 2 ? kz : L - kz) * nkx]);
      }
    }
    inv_fft_swapped<T2, L>(v, xb, tw, t);
#pragma unroll
    for (int i = 0; i < G::E; ++i) {
      const int z = G::TL::in_index(t, i);
      if (i % G::R2 < G::R2 / 2) ib[z * CW + line] = v[i];
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tma_store4(&tm, col0 * C0S, ky, 0, b, ib);
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait0();
}

// ---- planar grids (h.planar, one occupied z plane z0): y fwd * H_hat2 * y inv
// in one pass, bufA[y < Ny][col] -> bufC[y < Ny, occupied][col].  With all
// sources and potentials on z0 the z transform pair collapses exactly and the
// padded 3-D convolution is the padded 2-D one with the dz = 0 kernel slice,
// whose spectrum H_hat2[ky][kx] (scaled by 1/(4 N_x N_y)) is generated per
// frequency (spectrum.cu, planar plan).  The CTA's slab of H_hat2 (the octant
// rows ky <= N_y of its CW/4 kx, mirrored on read) is staged in shared memory
// while the forward transform runs.
// Columns col = nc kx + c (h.nc = 3 on planar grids: channels x, y, rho).
template <typename T, int L>
__global__ void __launch_bounds__(256, 2) k_yconv_plane(HotDev h) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using G = PassGeom<T, L>;
  const int line = threadIdx.x % G::NL, t = threadIdx.x / G::NL;
  const int W = h.W, Nx = h.Nx, Ny = h.Ny, nc = h.nc;
  const ColTile ct = col_tile<T, L>(line, W);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* xb = tw + L + line * G::XB;
  T2* hs = tw + L + (size_t)G::NL * G::XB;          // [ky <= Ny][kx - kx0]
  const int ja = blockIdx.x * ct.CW;                 // first column of the tile
  const int kx0 = h.kx0 + ja / nc;
  const int nkx = (ja + ct.CW - 1) / nc - ja / nc + 1;
  const int b = blockIdx.z;
  const T2* __restrict__ Hb = (const T2*)h.Hoct + b * h.sH;
  // the plane's occupied rows (they gate the loads) by plain loads; the
  // twiddles and the H_hat2 slab by cp.async (two commit groups), landing
  // behind the input loads and the forward transform respectively
  uint8_t* occ = reinterpret_cast<uint8_t*>(hs + (L / 2 + 1) * nkx);
  for (int y = threadIdx.x; y < Ny; y += blockDim.x) occ[y] = h.line_occ[(int64_t)h.zplane0 * Ny + y];
  for (int i = threadIdx.x; i < L; i += blockDim.x) cp_async(tw + i, (const T2*)h.twy_tab + i);
  asm volatile("cp.async.commit_group;\n" ::);
  for (int i = threadIdx.x; i < (L / 2 + 1) * nkx; i += blockDim.x) {
    const int ky = i / nkx, kx = kx0 + i % nkx;
    cp_async(hs + i, Hb + (int64_t)ky * (Nx + 1) + (kx <= Nx ? kx : 2 * Nx - kx));
  }
  asm volatile("cp.async.commit_group;\n" ::);
  __syncthreads();
  const bool act = ct.rsub == 0;   // one plane: the column tile's first row set only
  const int64_t col = ja + ct.w;
  const int kxl = (ja + ct.w) / nc - ja / nc;
  // per-element offsets in 32 bits (one slot's plane: Ny W < 2^31)
  const T2* __restrict__ in = (const T2*)h.bufA + b * h.sA + col;
  // this thread's occupied rows as a bit mask (the loads and the stores use
  // the same rows): one shared-memory byte read per row, once
  static_assert(G::E <= 64, "row mask");
  uint64_t om = 0;
#pragma unroll
  for (int i = 0; i < G::E; ++i)
    if (i % G::R2 < G::R2 / 2 && occ[G::TL::in_index(t, i)]) om |= 1ull << i;
  T2 v[G::E];
#pragma unroll
  for (int i = 0; i < G::E; ++i) {   // y < Ny = L/2  <=>  n2 < R2/2; unoccupied rows are zero
    const int y = G::TL::in_index(t, i);
    v[i] = (act && ((om >> i) & 1)) ? in[y * W] : mk<T2>(0, 0);
  }
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");   // the twiddles
  __syncthreads();
  fwd_fft<T2, L>(v, xb, tw, t);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");   // the slab
  __syncthreads();
  {
    const T2* hl = hs + kxl;
#pragma unroll
    for (int i = 0; i < G::E; ++i) {
      const int ky = TwoLevel<G::R2, G::R1>::in_index(t, i);
      v[i] = cmul(v[i], hl[(ky <= L / 2 ? ky : L - ky) * nkx]);
    }
  }
  inv_fft_swapped<T2, L>(v, xb, tw, t);
  if (!act) return;
  T2* __restrict__ out = (T2*)h.bufC + b * h.sA + col;
#pragma unroll
  for (int i = 0; i < G::E; ++i)
    if ((om >> i) & 1) out[G::TL::in_index(t, i) * W] = v[i];
}

// ---- fused y fwd -> (z fwd * H_hat * z inv) -> y inv for short y and z
// transforms (2 N_y, 2 N_z <= 32): one CTA owns a tile of TW grid columns
// (col = 4 kx + channel) and all (y, z) of them in shared memory, every line
// transform is one thread's register DFT.  bufA[z][y < Ny][col] -> bufC[z][y
// occupied][col]; the padded intermediate never leaves the SM.
template <typename T, int LY, int LZ> struct YZGeom {
  static constexpr int TW = sizeof(T) == 4 ? 32 : 16;   // columns per CTA
  static constexpr int NT = 128;
  // only z < N_z = LZ/2 is ever stored (inputs there, outputs cropped there)
  static constexpr size_t SMEM = sizeof(typename CT<T>::T2) * (size_t)(LZ / 2) * LY * TW;
};

template <typename T, int LY, int LZ, bool CURL = false>
__global__ void __launch_bounds__(128, sizeof(T) == 4 ? 4 : 2) k_yzconv(HotDev h) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using G = YZGeom<T, LY, LZ>;
  constexpr int TW = G::TW, NT = G::NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* S = reinterpret_cast<T2*>(smem_raw);   // [z < Nz][ky < LY][TW]
  const int Nx = h.Nx, Ny = h.Ny, Nz = h.Nz, W = h.W;
  const int b = blockIdx.y;
  const int col0 = blockIdx.x * TW;
  const T2* __restrict__ A = (const T2*)h.bufA + b * h.sA;
  T2* __restrict__ C = (T2*)h.bufC + b * h.sA;
  // phase 1: y forward of the z < Nz lines (zero for unoccupied planes)
  for (int it = threadIdx.x; it < Nz * TW; it += NT) {
    const int z = it / TW, w = it % TW;
    T2 v[LY];
    const bool occ = h.zocc[z];
#pragma unroll
    for (int y = 0; y < LY; ++y)
      v[y] = (occ && y < Ny) ? A[((int64_t)z * Ny + y) * W + col0 + w] : mk<T2>(0, 0);
    dftr<T2, LY, false>(v);
#pragma unroll
    for (int ky = 0; ky < LY; ++ky) S[(z * LY + ky) * TW + w] = v[ky];
  }
  __syncthreads();
  // phase 2: z forward, spectrum multiply, z inverse (z < Nz kept)
  const T2* __restrict__ Hb = (const T2*)h.Hoct + b * h.sH;
  if constexpr (CURL) {
    // per (ky, kx): the three current channels' z lines, Phi = G_hat x J_hat
    // (G_hat_a odd along a: sign change past N_a), channel 3 -> 0
    const int64_t noct = (int64_t)(Nx + 1) * (Ny + 1) * (Nz + 1);
    for (int it = threadIdx.x; it < LY * (TW / 4); it += NT) {
      const int ky = it / (TW / 4), w0 = 4 * (it % (TW / 4));
      const int kx = h.kx0 + ((col0 + w0) >> 2);
      const int kxf = kx <= Nx ? kx : 2 * Nx - kx, kyf = ky <= Ny ? ky : 2 * Ny - ky;
      const T sx = kx > Nx ? T(-1) : T(1), sy = ky > Ny ? T(-1) : T(1);
      T2 J[3][LZ];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int z = 0; z < LZ; ++z) J[c][z] = z < Nz ? S[(z * LY + ky) * TW + w0 + c] : mk<T2>(0, 0);
        dftr<T2, LZ, false>(J[c]);
      }
      const T2* hl = Hb + (int64_t)kyf * (Nz + 1) * (Nx + 1) + kxf;
#pragma unroll
      for (int kz = 0; kz < LZ; ++kz) {
        const int kzf = kz <= Nz ? kz : 2 * Nz - kz;
        const T sz = kz > Nz ? T(-1) : T(1);
        const T2 a0 = hl[(int64_t)kzf * (Nx + 1)], a1 = hl[noct + (int64_t)kzf * (Nx + 1)],
                 a2 = hl[2 * noct + (int64_t)kzf * (Nx + 1)];
        const T2 gx = mk<T2>(sx * a0.x, sx * a0.y), gy = mk<T2>(sy * a1.x, sy * a1.y),
                 gz = mk<T2>(sz * a2.x, sz * a2.y);
        const T2 px = csub(cmul(gy, J[2][kz]), cmul(gz, J[1][kz]));
        const T2 py = csub(cmul(gz, J[0][kz]), cmul(gx, J[2][kz]));
        const T2 pz = csub(cmul(gx, J[1][kz]), cmul(gy, J[0][kz]));
        J[0][kz] = px;
        J[1][kz] = py;
        J[2][kz] = pz;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        dftr<T2, LZ, true>(J[c]);
#pragma unroll
        for (int z = 0; z < LZ; ++z)
          if (z < Nz) S[(z * LY + ky) * TW + w0 + c] = J[c][z];
      }
#pragma unroll
      for (int z = 0; z < LZ; ++z)
        if (z < Nz) S[(z * LY + ky) * TW + w0 + 3] = mk<T2>(0, 0);
    }
  } else
  for (int it = threadIdx.x; it < LY * TW; it += NT) {
    const int ky = it / TW, w = it % TW;
    const int kx = h.kx0 + ((col0 + w) >> 2);
    const int kxf = kx <= Nx ? kx : 2 * Nx - kx;
    const int kyf = ky <= Ny ? ky : 2 * Ny - ky;
    T2 v[LZ];
#pragma unroll
    for (int z = 0; z < LZ; ++z) v[z] = z < Nz ? S[(z * LY + ky) * TW + w] : mk<T2>(0, 0);
    dftr<T2, LZ, false>(v);
    const T2* hl = Hb + (int64_t)kyf * (Nz + 1) * (Nx + 1) + kxf;
#pragma unroll
    for (int kz = 0; kz < LZ; ++kz) {
      const int kzf = kz <= Nz ? kz : 2 * Nz - kz;
      v[kz] = cmul(v[kz], hl[(int64_t)kzf * (Nx + 1)]);
    }
    dftr<T2, LZ, true>(v);
#pragma unroll
    for (int z = 0; z < LZ; ++z)
      if (z < Nz) S[(z * LY + ky) * TW + w] = v[z];
  }
  __syncthreads();
  // phase 3: y inverse of the occupied planes, occupied lines stored
  for (int it = threadIdx.x; it < Nz * TW; it += NT) {
    const int z = it / TW, w = it % TW;
    if (!h.zocc[z]) continue;
    T2 v[LY];
#pragma unroll
    for (int ky = 0; ky < LY; ++ky) v[ky] = S[(z * LY + ky) * TW + w];
    dftr<T2, LY, true>(v);
    const uint8_t* occ = h.line_occ + (int64_t)z * Ny;
#pragma unroll
    for (int y = 0; y < LY; ++y)
      if (y < Ny && occ[y]) C[((int64_t)z * Ny + y) * W + col0 + w] = v[y];
  }
}

// ------------------------------------------------------------------ S4 + S5
// Row groups (NearGroups): R spatially ordered testing functions share one
// sorted union of their stencil nodes (interpolation W = P^T) and one
// sorted union of their near columns (C = L_s,NR - L_s,P, eq:LAIMx P:283);
// each union entry carries R coefficient tuples, so a potential row (4
// channels x BB columns) or an x row (BB columns) is read once for R rows.
//
// One CTA walks a contiguous range of whole groups as a stream of chunks
// (NearChunks): per group its W (interpolation) chunks, then its C (near)
// chunks.  The dense coefficient blocks -- the HBM stream -- are moved by the
// TMA bulk-copy engine into a ring of D+1 shared-memory stages, D chunks ahead,
// completion tracked by one mbarrier per stage; the row indices (two D ahead)
// and chunk descriptors (three D ahead) ride on the same barriers.  The
// gathered rows -- x rows (C) and potential rows (W), L2-resident -- are
// loaded straight into registers one chunk ahead (ping-pong register buffers),
// so their latency overlaps the previous chunk's arithmetic.  Lanes: group g of
// LG lanes covers V columns per lane (16-byte loads); the NLG lane groups of
// the CTA stride the chunk's entries.  At a group's last chunk the partial sums
// are reduced in a fixed order (shuffles within the warp, then shared memory)
// and combined: y = -j w mu0 (y^A - k0^-2 y^rho) (eq:EFIEAIMx P:288), or the
// unscaled parts y^A and -y^rho (PARTS).
template <typename T2, int V> struct VecT;
template <> struct VecT<float2, 1> { using type = float2; };
template <> struct VecT<float2, 2> { using type = float4; };
template <> struct VecT<double2, 1> { using type = double2; };

template <typename T, int R, int BB, bool PARTS> struct NearCfg {
  using T2 = typename CT<T>::T2;
  static constexpr int NT = 128;                      // threads per CTA
  static constexpr int S = (int)sizeof(T2);           // complex bytes
  // entries per C / W chunk (at most; near_chc / near_chw, halved for 32 columns)
  static constexpr int CHC = (BB >= 32 ? 512 : 1024) / S, CHW = (BB >= 32 ? 128 : 256) / S;
  static constexpr int COEFB = CHC * R * S;           // coefficient bytes (C: R pairs; W: R real4 = 2 S per entry)
  static constexpr int STB = COEFB + CHC * 4 + 16;    // stage: one chunk payload (NearChunks)
  static constexpr int D = kNearD;                    // pipeline depth (chunks)
  static constexpr int NDS = D + 1, NDD = D + 1;      // stage / descriptor slots
  static constexpr int V = (S == 8 && BB >= 2) ? 2 : 1;
  static constexpr int LG = BB / V, NG = 32 / LG, NLG = (NT / 32) * NG;
  static constexpr int NPC = (CHC + NLG - 1) / NLG;   // C entries per lane group per chunk
  static constexpr int NPW = (CHW + NLG - 1) / NLG;   // W entries per lane group per chunk
  static constexpr int NBUF = NPC > 4 * NPW ? NPC : 4 * NPW;   // row loads in flight per lane
  static constexpr int NA = (PARTS ? 2 : 1) * R * V;  // complex accumulators: [part][r][v]
  static constexpr int NV = 2 * NA;                   // as reals
  // partial sums per (warp, lane of group 0), after a shuffle reduction over
  // the warp's NG lane groups (small shared footprint: 5 CTAs per SM fit at
  // every column count)
  static constexpr bool SHFL = true;
  static constexpr size_t REDB = (size_t)(SHFL ? (NT / 32) * LG : NT) * (NV + 1) * sizeof(T);
  static constexpr size_t OFF_RED = (size_t)NDS * STB;
  static constexpr size_t OFF_DESC = (OFF_RED + REDB + 15) / 16 * 16;
  static constexpr size_t OFF_BAR = OFF_DESC + NDD * 16;
  static constexpr size_t SMEM = OFF_BAR + NDS * 8;
};

template <typename T2, int V>
__device__ __forceinline__ void unpack(const typename VecT<T2, V>::type& u, T2* out) {
  if constexpr (V == 2) {
    out[0] = mk<T2>(u.x, u.y);
    out[1] = mk<T2>(u.z, u.w);
  } else {
    out[0] = u;
  }
}

template <typename T, int R, int BB, bool PARTS>
__global__ void __launch_bounds__(128, near_ctas_per_sm(sizeof(T) == 4, BB == 1, R))
    k_interp_near(HotDev h, const typename CT<T>::T2* __restrict__ xt,
                                                     typename CT<T>::T2* __restrict__ y0,
                                                     typename CT<T>::T2* __restrict__ y1, Combine cb) {
  pdl_wait();
  pdl_trigger();
  using K = NearCfg<T, R, BB, PARTS>;
  using T2 = typename CT<T>::T2;
  using T4 = typename CT<T>::T4;
  using VT = typename VecT<T2, K::V>::type;
  constexpr int NT = K::NT, V = K::V, LG = K::LG, NG = K::NG, NLG = K::NLG, NV = K::NV, NA = K::NA;
  constexpr int D = K::D, CHC = K::CHC, NPC = K::NPC;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* const sdata = smem;                                         // [NDS][STB]
  T* const red = reinterpret_cast<T*>(smem + K::OFF_RED);                    // partial sums
  int4* const sdesc = reinterpret_cast<int4*>(smem + K::OFF_DESC);           // [NDD]
  uint64_t* const bar = reinterpret_cast<uint64_t*>(smem + K::OFF_BAR);      // [NDS]
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int b0 = (lane % LG) * V, g = lane / LG, lgid = wib * NG + g;
  const int32_t* __restrict__ cta_ptr = BB == 1 ? h.cta_ptr1 : h.cta_ptr;
  const int c0 = cta_ptr[blockIdx.x], nch = cta_ptr[blockIdx.x + 1] - c0;
  if (nch <= 0) return;
  const int4* __restrict__ chunks = reinterpret_cast<const int4*>(h.chunks) + c0;
  const int nc = h.nc;                            // stored channels: 4, or 3 (x, y, rho) on planar grids
  const int64_t ns = (int64_t)h.batch * nc;       // phi node stride (complex): [node][channel][slot]
  const T2* __restrict__ phi = (const T2*)h.phi + b0;
  const T2* __restrict__ xr = xt + b0;
  T be[V];
#pragma unroll
  for (int v = 0; v < V; ++v) be[v] = PARTS ? T(0) : (T)cb.beta[b0 + v];   // 0 for b >= B
  T2 acc[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) acc[i] = mk<T2>(0, 0);
  const T2 nbe2 = mk<T2>(-be[0], V == 2 ? -be[V - 1] : T(0));   // (-beta_b0, -beta_b0+1)

  // coefficient bytes of a chunk
  auto coef_bytes = [&](const int4& d) -> int { return d.w * R * ((d.y & 1) ? K::S : 2 * K::S); };
  // ONE bulk copy moves chunk j's payload (coefficients, row indices, the
  // descriptor of chunk j + D) into stage j % NDS, completing on bar[j % NDS]
  // (thread 0; d = chunk j's descriptor, recorded for the compute)
  auto issue = [&](int j, const int4& d) {
    uint64_t* bj = bar + j % K::NDS;
    const uint32_t bytes = (uint32_t)(coef_bytes(d) + ((4 * d.w + 15) & ~15) + 16);
    sdesc[j % K::NDD] = d;
    mbar_arrive_expect_tx(bj, bytes);
    bulk_g2s(sdata + (j % K::NDS) * K::STB, h.payload + (int64_t)d.z * 16, bytes, bj);
  };

  // prologue: barriers; descriptors 0..D-1 by plain loads; chunks 0..D-1 in flight
  if (tid < K::NDS) mbar_init(bar + tid, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  if (tid == 0)
    for (int j = 0; j < D && j < nch; ++j) issue(j, chunks[j]);
  __syncthreads();

  // gathered rows of a landed chunk into registers (all loads issued before any
  // use): C: x rows of entries lgid + i NLG; W: the 4 channel rows of entries
  // lgid + i NLG
  auto gather = [&](const int4& d, const unsigned char* stg, VT* b) {
    const int* ix = reinterpret_cast<const int*>(stg + coef_bytes(d));
    if (d.y & 1) {
#pragma unroll
      for (int i = 0; i < K::NPC; ++i) {
        const int e = lgid + i * NLG;
        if (e < d.w) b[i] = __ldg((const VT*)(xr + (int64_t)ix[e] * BB));
      }
    } else {
#pragma unroll
      for (int i = 0; i < K::NPW; ++i) {
        const int e = lgid + i * NLG;
        if (e < d.w) {
          const T2* pr = phi + (int64_t)ix[e] * ns;
#pragma unroll
          for (int c = 0; c < 4; ++c)   // nc = 3: phi_z is not stored (Lambda^z = 0), slot 2 holds rho
            if (c < nc) b[4 * i + c] = __ldg((const VT*)(pr + (int64_t)c * h.batch));
        }
      }
    }
  };
  // Single column (few registers per lane): the rows of chunk k + 1 are
  // gathered while chunk k computes, so their L2 latency is off the per-chunk
  // chain (wait -> indices -> gather -> arithmetic -> block barrier).
  constexpr bool PRE = BB == 1;
  VT buf[K::NBUF];
  [[maybe_unused]] VT nbuf[PRE ? K::NBUF : 1];
  if constexpr (PRE) {
    mbar_wait(bar, 0u);
    gather(sdesc[0], sdata, nbuf);
  }
  for (int k = 0; k < nch; ++k) {
    // chunk k's payload (with the descriptor of chunk k + D) has landed
    if constexpr (!PRE) mbar_wait(bar + k % K::NDS, (uint32_t)(k / K::NDS) & 1u);
    const int4 d = sdesc[k % K::NDD];
    const unsigned char* stg = sdata + (k % K::NDS) * K::STB;
    if (tid == 0 && k + D < nch)
      issue(k + D, *reinterpret_cast<const int4*>(stg + coef_bytes(d) + ((4 * d.w + 15) & ~15)));
    if constexpr (PRE) {
#pragma unroll
      for (int i = 0; i < K::NBUF; ++i) buf[i] = nbuf[i];
      if (k + 1 < nch) {
        mbar_wait(bar + (k + 1) % K::NDS, (uint32_t)((k + 1) / K::NDS) & 1u);
        gather(sdesc[(k + 1) % K::NDD], sdata + ((k + 1) % K::NDS) * K::STB, nbuf);
      }
    } else {
      gather(d, stg, buf);
    }
    if (d.y & 1) {   // near correction: pairs [e][R]
      const T2* __restrict__ cf = (const T2*)stg;
#pragma unroll
      for (int i = 0; i < K::NPC; ++i) {
        const int e = lgid + i * NLG;
        if (e >= d.w) break;
        T2 xv[V];
        unpack<T2, V>(buf[i], xv);
        T2 cv[R];
        if constexpr (K::S == 8) {
#pragma unroll
          for (int q = 0; q < R / 2; ++q) {
            const float4 f = reinterpret_cast<const float4*>(cf + e * R)[q];
            cv[2 * q] = mk<T2>(f.x, f.y);
            cv[2 * q + 1] = mk<T2>(f.z, f.w);
          }
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) cv[r] = cf[e * R + r];
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if constexpr (PARTS) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
              axpy(acc[r * V + v], cv[r].x, xv[v]);
              axpy(acc[(R + r) * V + v], cv[r].y, xv[v]);
            }
          } else if constexpr (K::S == 8 && V == 2) {
            // (ce_0, ce_1) = C_A - beta_b C_rho for both columns: one FFMA2
            const T2 ce = ffma2(nbe2, mk<T2>(cv[r].y, cv[r].y), mk<T2>(cv[r].x, cv[r].x));
            axpy(acc[r * V], ce.x, xv[0]);
            axpy(acc[r * V + 1], ce.y, xv[1]);
          } else {
#pragma unroll
            for (int v = 0; v < V; ++v) axpy(acc[r * V + v], cv[r].x - be[v] * cv[r].y, xv[v]);
          }
        }
      }
    } else {         // interpolation: weights [e][R] real4
#pragma unroll
      for (int i = 0; i < K::NPW; ++i) {
      const int e = lgid + i * NLG;
      if (e >= d.w) break;
      const T4* __restrict__ wf = (const T4*)stg + e * R;
      T2 pv[4][V];
#pragma unroll
      for (int c = 0; c < 4; ++c) unpack<T2, V>(buf[4 * i + (c == 3 && nc == 3 ? 2 : c)], pv[c]);   // rho
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const T4 w = wf[r];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          T2& a = acc[r * V + v];
          axpy(a, w.x, pv[0][v]);
          axpy(a, w.y, pv[1][v]);
          if (nc == 4) axpy(a, w.z, pv[2][v]);
          if constexpr (PARTS) axpy(acc[(R + r) * V + v], w.w, pv[3][v]);
          else axpy(a, -be[v] * w.w, pv[3][v]);
        }
      }
      }
    }
    if (d.y & 4) {   // last chunk of group d.x: fixed-order reduction + combine
      int nsrc;      // partial-sum rows per output lane
      if constexpr (K::SHFL) {
#pragma unroll
        for (int o = LG; o < 32; o <<= 1)
#pragma unroll
          for (int i = 0; i < NA; ++i) {
            acc[i].x += __shfl_xor_sync(0xffffffffu, acc[i].x, o);
            acc[i].y += __shfl_xor_sync(0xffffffffu, acc[i].y, o);
          }
        if (g == 0)
#pragma unroll
          for (int i = 0; i < NA; ++i) {
            red[(wib * LG + lane) * (NV + 1) + 2 * i] = acc[i].x;
            red[(wib * LG + lane) * (NV + 1) + 2 * i + 1] = acc[i].y;
          }
        nsrc = NT / 32;
      } else {
#pragma unroll
        for (int i = 0; i < NA; ++i) {
          red[tid * (NV + 1) + 2 * i] = acc[i].x;
          red[tid * (NV + 1) + 2 * i + 1] = acc[i].y;
        }
        nsrc = NLG;
      }
#pragma unroll
      for (int i = 0; i < NA; ++i) acc[i] = mk<T2>(0, 0);
      __syncthreads();
      const int32_t* gr = h.grp_rows + (int64_t)d.x * R;
      for (int o = tid; o < LG * NV; o += NT) {
        const int lb = o / NV, i = o % NV;
        T sum = T(0);
        // source row j of output lane lb: SHFL: warp j's lane lb; else lane group j
        for (int j = 0; j < nsrc; ++j) {
          const int row = K::SHFL ? j * LG + lb : (j / NG) * 32 + (j % NG) * LG + lb;
          sum += red[row * (NV + 1) + i];
        }
        const int comp = i & 1, v = (i >> 1) % V, r = (i / (2 * V)) % R, part = i / (2 * V * R);
        const int m = gr[r];
        if (m < 0) continue;
        if constexpr (PARTS) {
          T2* y = part ? y1 : y0;
          if (y) reinterpret_cast<T*>(y + m)[comp] = part ? -sum : sum;
        } else {
          const int b = lb * V + v;
          if (b < cb.B) {   // (j alpha) u: re = -alpha u.im, im = alpha u.re
            const T al = (T)cb.alpha_im[b];
            T* yy = reinterpret_cast<T*>(y0 + (int64_t)b * cb.ystride + m);
            if (comp == 0) yy[1] = al * sum;
            else yy[0] = -al * sum;
          }
        }
      }
    }
    __syncthreads();   // stage and descriptor slots of chunk k are refilled next
  }
}

// shared-memory layout of k_interp_near1: NearCfg<float, 8, 1, PARTS>'s with the
// stage sized for the context's chunk length (HALF: 8 CTAs per SM fit)
template <bool PARTS, bool HALF> struct Near1Smem {
  using K = NearCfg<float, 8, 1, PARTS>;
  static constexpr int CH = K::CHC / (HALF ? 2 : 1);
  static constexpr int STB = CH * 8 * 8 + CH * 4 + 16;
  static constexpr size_t OFF_RED = (size_t)K::NDS * STB;
  static constexpr size_t OFF_DESC = (OFF_RED + K::REDB + 15) / 16 * 16;
  static constexpr size_t OFF_BAR = OFF_DESC + K::NDD * 16;
  static constexpr size_t SMEM = OFF_BAR + K::NDS * 8;
};

// S4+S5, ONE column, c64, R = 8 rows per group (the single matvec of a GMRES
// iteration: HBM-bound on the coefficient stream).  The same chunk payload
// and TMA ring as k_interp_near, but the lanes split an entry's rows instead
// of taking one entry each: C chunks: 4 lanes per entry, lane q reads the
// 16-byte word of rows 2q, 2q+1 ((C_A, C_rho) pairs); W chunks: 8 lanes per
// entry, lane r reads row r's real4 weight.  Consecutive lanes read consecutive
// 16-byte words of the stage, so the shared-memory reads are conflict-free
// (one entry per lane strides them by 64 / 128 bytes: 4- / 8-way conflicts,
// the shared pipe at 65% and the limiter, profiles/r2h_near1.md), every
// thread has work on the short chunks of 32-slot contexts, and a group ends
// with 16 shuffles per lane instead of 80.  The gathered x / potential values
// of chunk k + 1 load while chunk k computes.
template <bool PARTS, bool HALF>
__global__ void __launch_bounds__(128, near1_ctas_per_sm(HALF))
    k_interp_near1(HotDev h, const float2* __restrict__ xt, float2* __restrict__ y0, float2* __restrict__ y1,
                   Combine cb) {
  pdl_wait();
  pdl_trigger();
  using K = NearCfg<float, 8, 1, PARTS>;
  constexpr int R = 8, NT = K::NT, D = K::D, NP = PARTS ? 2 : 1;
  // HALF: the context holds 32 batch slots, its payload chunks are half length
  // (near_chc / near_chw)
  constexpr int PC = K::CHC / 32 / (HALF ? 2 : 1);   // C passes: 32 entries per pass
  constexpr int PW = K::CHW / 16 / (HALF ? 2 : 1);   // W passes: 16 entries per pass
  constexpr int NB = PC > 4 * PW ? PC : 4 * PW;
  using SM = Near1Smem<PARTS, HALF>;
  constexpr int STB = SM::STB;   // stage: one (half-length) chunk payload
  static_assert(K::CHC % 32 == 0 && K::CHW % 16 == 0 && NT == 128, "lane mapping");
  static_assert(K::REDB >= (size_t)(NT / 32) * NP * R * sizeof(float2), "partial sums");
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* const sdata = smem;                                         // [NDS][STB]
  float2* const red = reinterpret_cast<float2*>(smem + SM::OFF_RED);          // [warp][part][R]
  int4* const sdesc = reinterpret_cast<int4*>(smem + SM::OFF_DESC);           // [NDD]
  uint64_t* const bar = reinterpret_cast<uint64_t*>(smem + SM::OFF_BAR);      // [NDS]
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int c0 = h.cta_ptr1[blockIdx.x], nch = h.cta_ptr1[blockIdx.x + 1] - c0;
  if (nch <= 0) return;
  const int4* __restrict__ chunks = reinterpret_cast<const int4*>(h.chunks) + c0;
  const int nc = h.nc;                            // stored channels: 4, or 3 (x, y, rho) on planar grids
  const int64_t ns = (int64_t)h.batch * nc;       // phi node stride (complex): [node][channel][slot]
  const float2* __restrict__ phi = (const float2*)h.phi;
  const float be = PARTS ? 0.f : (float)cb.beta[0];

  auto coef_bytes = [&](const int4& d) -> int { return d.w * R * ((d.y & 1) ? 8 : 16); };
  auto issue = [&](int j, const int4& d) {   // as in k_interp_near
    uint64_t* bj = bar + j % K::NDS;
    const uint32_t bytes = (uint32_t)(coef_bytes(d) + ((4 * d.w + 15) & ~15) + 16);
    sdesc[j % K::NDD] = d;
    mbar_arrive_expect_tx(bj, bytes);
    bulk_g2s(sdata + (j % K::NDS) * STB, h.payload + (int64_t)d.z * 16, bytes, bj);
  };
  if (tid < K::NDS) mbar_init(bar + tid, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  if (tid == 0)
    for (int j = 0; j < D && j < nch; ++j) issue(j, chunks[j]);
  __syncthreads();

  const int ec = tid >> 2, qc = tid & 3;   // C: entry of pass 0, row pair
  const int ew = tid >> 3, rw = tid & 7;   // W: entry of pass 0, row
  auto gather = [&](const int4& d, const unsigned char* stg, float2* b) {
    const int* ix = reinterpret_cast<const int*>(stg + coef_bytes(d));
    if (d.y & 1) {
#pragma unroll
      for (int i = 0; i < PC; ++i) {
        const int e = ec + 32 * i;
        if (e < d.w) b[i] = __ldg(xt + ix[e]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < PW; ++i) {
        const int e = ew + 16 * i;
        if (e < d.w) {
          const float2* pr = phi + (int64_t)ix[e] * ns;
#pragma unroll
          for (int c = 0; c < 4; ++c)   // nc = 3: phi_z is not stored (Lambda^z = 0), slot 2 holds rho
            if (c < nc) b[4 * i + c] = __ldg(pr + (int64_t)c * h.batch);
        }
      }
    }
  };

  float2 aC[2 * NP], aW[NP];   // C: [part][row 2 qc + j]; W: [part] of row rw
#pragma unroll
  for (int j = 0; j < 2 * NP; ++j) aC[j] = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < NP; ++j) aW[j] = make_float2(0.f, 0.f);
  // (swapping two register buffers in a loop unrolled by two instead of the
  // copy was measured slower: cfg3 0.091 -> 0.099 ms)
  float2 buf[NB], nbuf[NB];
  mbar_wait(bar, 0u);
  gather(sdesc[0], sdata, nbuf);
  for (int k = 0; k < nch; ++k) {
    const int4 d = sdesc[k % K::NDD];
    const unsigned char* stg = sdata + (k % K::NDS) * STB;
    if (tid == 0 && k + D < nch)
      issue(k + D, *reinterpret_cast<const int4*>(stg + coef_bytes(d) + ((4 * d.w + 15) & ~15)));
#pragma unroll
    for (int i = 0; i < NB; ++i) buf[i] = nbuf[i];
    if (k + 1 < nch) {
      mbar_wait(bar + (k + 1) % K::NDS, (uint32_t)((k + 1) / K::NDS) & 1u);
      gather(sdesc[(k + 1) % K::NDD], sdata + ((k + 1) % K::NDS) * STB, nbuf);
    }
    if (d.y & 1) {   // near correction: [e][R] (C_A, C_rho) pairs
      const float4* __restrict__ cf = reinterpret_cast<const float4*>(stg);
#pragma unroll
      for (int i = 0; i < PC; ++i) {
        const int e = ec + 32 * i;
        if (e >= d.w) break;
        const float4 f = cf[e * 4 + qc];
        const float2 x = buf[i];
        if constexpr (PARTS) {
          axpy(aC[0], f.x, x);
          axpy(aC[2], f.y, x);
          axpy(aC[1], f.z, x);
          axpy(aC[3], f.w, x);
        } else {
          axpy(aC[0], f.x - be * f.y, x);
          axpy(aC[1], f.z - be * f.w, x);
        }
      }
    } else {         // interpolation: [e][R] real4 weights
      const float4* __restrict__ wf = reinterpret_cast<const float4*>(stg);
#pragma unroll
      for (int i = 0; i < PW; ++i) {
        const int e = ew + 16 * i;
        if (e >= d.w) break;
        const float4 w = wf[e * 8 + rw];
        axpy(aW[0], w.x, buf[4 * i]);
        axpy(aW[0], w.y, buf[4 * i + 1]);
        if (nc == 4) axpy(aW[0], w.z, buf[4 * i + 2]);
        const float2 rho = nc == 4 ? buf[4 * i + 3] : buf[4 * i + 2];
        if constexpr (PARTS) axpy(aW[1], w.w, rho);
        else axpy(aW[0], -be * w.w, rho);
      }
    }
    if (d.y & 4) {   // last chunk of group d.x: fixed-order reduction + combine
#pragma unroll
      for (int o = 4; o < 32; o <<= 1)
#pragma unroll
        for (int j = 0; j < 2 * NP; ++j) {
          aC[j].x += __shfl_xor_sync(0xffffffffu, aC[j].x, o);
          aC[j].y += __shfl_xor_sync(0xffffffffu, aC[j].y, o);
        }
#pragma unroll
      for (int o = 8; o < 32; o <<= 1)
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          aW[j].x += __shfl_xor_sync(0xffffffffu, aW[j].x, o);
          aW[j].y += __shfl_xor_sync(0xffffffffu, aW[j].y, o);
        }
      // row r = lane (< 8): its C sums sit in lanes with qc = r >> 1, slot r & 1
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const int src = (lane >> 1) & 3;
        const float a0x = __shfl_sync(0xffffffffu, aC[2 * p].x, src), a0y = __shfl_sync(0xffffffffu, aC[2 * p].y, src);
        const float a1x = __shfl_sync(0xffffffffu, aC[2 * p + 1].x, src), a1y = __shfl_sync(0xffffffffu, aC[2 * p + 1].y, src);
        if (lane < R)
          red[(wib * NP + p) * R + lane] =
              make_float2(aW[p].x + ((lane & 1) ? a1x : a0x), aW[p].y + ((lane & 1) ? a1y : a0y));
      }
#pragma unroll
      for (int j = 0; j < 2 * NP; ++j) aC[j] = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < NP; ++j) aW[j] = make_float2(0.f, 0.f);
      __syncthreads();
      if (tid < NP * R) {
        const int p = tid / R, r = tid % R;
        float2 sum = make_float2(0.f, 0.f);
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) {
          const float2 v = red[(w * NP + p) * R + r];
          sum.x += v.x;
          sum.y += v.y;
        }
        const int m = h.grp_rows[(int64_t)d.x * R + r];
        if (m >= 0) {
          if constexpr (PARTS) {
            float2* y = p ? y1 : y0;
            if (y) y[m] = p ? make_float2(-sum.x, -sum.y) : sum;
          } else {   // (j alpha) u: re = -alpha u.im, im = alpha u.re
            const float al = (float)cb.alpha_im[0];
            y0[m] = make_float2(-al * sum.y, al * sum.x);
          }
        }
      }
    }
    __syncthreads();   // stage and descriptor slots of chunk k are refilled next
  }
}

// S4+S5, ONE column, c64, R = 8, 32-slot contexts (half-length chunks): the
// warp-private form of k_interp_near1.  Each WARP walks its own contiguous
// range of whole groups (warp_ptr1) through its own 3-stage TMA ring and
// mbarriers: no block barrier anywhere, a group ends inside the warp (shuffles,
// lanes 0..7 store the 8 rows), and the per-chunk bookkeeping (wait,
// descriptor, refill) is paid once per chunk instead of once per warp and
// chunk.  A stage is refilled (chunk k + D, whose descriptor rides in chunk
// k's payload) right after the warp has consumed it.  Lanes: C chunks 4 lanes
// per entry (lane q: rows 2q, 2q+1), 8 entries per pass; W chunks 8 lanes per
// entry (lane r: row r), 4 entries per pass; a chunk's gathers are all issued
// before its arithmetic.
struct Near1W {
  static constexpr int NT = 128, NW = NT / 32, PER_SM = 4;
  static constexpr int CH = 64, CW = 16;                 // near_chc / near_chw at 32 slots
  static constexpr int STB = CH * 8 * 8 + CH * 4 + 16;   // one chunk payload
  static constexpr int NS = kNearD;                      // stages per warp
  static_assert(CH == near_chc(true, 32) && CW == near_chw(true, 32), "chunk lengths of 32-slot c64 contexts");
  static constexpr size_t OFF_DESC = (size_t)NW * NS * STB;
  static constexpr size_t OFF_BAR = OFF_DESC + (size_t)NW * NS * 16;
  static constexpr size_t SMEM = OFF_BAR + (size_t)NW * NS * 8;
};

template <bool PARTS>
__global__ void __launch_bounds__(Near1W::NT, Near1W::PER_SM)
    k_interp_near1w(HotDev h, const float2* __restrict__ xt, float2* __restrict__ y0, float2* __restrict__ y1,
                    Combine cb) {
  pdl_wait();
  pdl_trigger();
  using K = Near1W;
  constexpr int R = 8, D = kNearD, NS = K::NS, STB = K::STB, NP = PARTS ? 2 : 1;
  constexpr int PC = K::CH / 8, PW = K::CW / 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* const sdata = smem + (size_t)wib * NS * STB;                         // [NS][STB]
  int4* const sdesc = reinterpret_cast<int4*>(smem + K::OFF_DESC) + wib * NS;         // [NS]
  uint64_t* const bar = reinterpret_cast<uint64_t*>(smem + K::OFF_BAR) + wib * NS;    // [NS]
  const int wid = blockIdx.x * K::NW + wib;
  const int c0 = h.warp_ptr1[wid], nch = h.warp_ptr1[wid + 1] - c0;
  if (nch <= 0) return;
  const int4* __restrict__ chunks = reinterpret_cast<const int4*>(h.chunks) + c0;
  const int nc = h.nc;
  const int64_t ns = (int64_t)h.batch * nc;
  const float2* __restrict__ phi = (const float2*)h.phi;
  const float be = PARTS ? 0.f : (float)cb.beta[0];
  const float al = (float)cb.alpha_im[0];

  auto coef_bytes = [&](const int4& d) -> int { return d.w * R * ((d.y & 1) ? 8 : 16); };
  auto issue = [&](int j, const int4& d) {   // lane 0
    uint64_t* bj = bar + j % NS;
    const uint32_t bytes = (uint32_t)(coef_bytes(d) + ((4 * d.w + 15) & ~15) + 16);
    sdesc[j % NS] = d;
    mbar_arrive_expect_tx(bj, bytes);
    bulk_g2s(sdata + (j % NS) * STB, h.payload + (int64_t)d.z * 16, bytes, bj);
  };
  if (lane == 0) {
    for (int j = 0; j < NS; ++j) mbar_init(bar + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int j = 0; j < D && j < nch; ++j) issue(j, chunks[j]);
  }
  __syncwarp();

  const int ec = lane >> 2, qc = lane & 3;   // C: entry of pass 0, row pair
  const int ew = lane >> 3, rw = lane & 7;   // W: entry of pass 0, row
  float2 aC[2 * NP], aW[NP];
#pragma unroll
  for (int j = 0; j < 2 * NP; ++j) aC[j] = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < NP; ++j) aW[j] = make_float2(0.f, 0.f);

  for (int k = 0; k < nch; ++k) {
    mbar_wait(bar + k % NS, (uint32_t)(k / NS) & 1u);
    const int4 d = sdesc[k % NS];
    const unsigned char* stg = sdata + (k % NS) * STB;
    const int* ix = reinterpret_cast<const int*>(stg + coef_bytes(d));
    const int4 dn = *reinterpret_cast<const int4*>(stg + coef_bytes(d) + ((4 * d.w + 15) & ~15));
    if (d.y & 1) {   // near correction: [e][R] (C_A, C_rho) pairs
      const float4* __restrict__ cf = reinterpret_cast<const float4*>(stg);
      float2 b[PC];
#pragma unroll
      for (int i = 0; i < PC; ++i) {
        const int e = ec + 8 * i;
        if (e < d.w) b[i] = __ldg(xt + ix[e]);
      }
#pragma unroll
      for (int i = 0; i < PC; ++i) {
        const int e = ec + 8 * i;
        if (e >= d.w) break;
        const float4 f = cf[e * 4 + qc];
        if constexpr (PARTS) {
          axpy(aC[0], f.x, b[i]);
          axpy(aC[2], f.y, b[i]);
          axpy(aC[1], f.z, b[i]);
          axpy(aC[3], f.w, b[i]);
        } else {
          axpy(aC[0], f.x - be * f.y, b[i]);
          axpy(aC[1], f.z - be * f.w, b[i]);
        }
      }
    } else {         // interpolation: [e][R] real4 weights
      const float4* __restrict__ wf = reinterpret_cast<const float4*>(stg);
      float2 b[4 * PW];
#pragma unroll
      for (int i = 0; i < PW; ++i) {
        const int e = ew + 4 * i;
        if (e < d.w) {
          const float2* pr = phi + (int64_t)ix[e] * ns;
#pragma unroll
          for (int c = 0; c < 4; ++c)   // nc = 3: slot 2 holds rho
            if (c < nc) b[4 * i + c] = __ldg(pr + (int64_t)c * h.batch);
        }
      }
#pragma unroll
      for (int i = 0; i < PW; ++i) {
        const int e = ew + 4 * i;
        if (e >= d.w) break;
        const float4 w = wf[e * 8 + rw];
        axpy(aW[0], w.x, b[4 * i]);
        axpy(aW[0], w.y, b[4 * i + 1]);
        if (nc == 4) axpy(aW[0], w.z, b[4 * i + 2]);
        const float2 rho = nc == 4 ? b[4 * i + 3] : b[4 * i + 2];
        if constexpr (PARTS) axpy(aW[1], w.w, rho);
        else axpy(aW[0], -be * w.w, rho);
      }
    }
    if (d.y & 4) {   // last chunk of group d.x: reduce inside the warp, combine, store
#pragma unroll
      for (int o = 4; o < 32; o <<= 1)
#pragma unroll
        for (int j = 0; j < 2 * NP; ++j) {
          aC[j].x += __shfl_xor_sync(0xffffffffu, aC[j].x, o);
          aC[j].y += __shfl_xor_sync(0xffffffffu, aC[j].y, o);
        }
#pragma unroll
      for (int o = 8; o < 32; o <<= 1)
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          aW[j].x += __shfl_xor_sync(0xffffffffu, aW[j].x, o);
          aW[j].y += __shfl_xor_sync(0xffffffffu, aW[j].y, o);
        }
      const int m = lane < R ? h.grp_rows[(int64_t)d.x * R + lane] : -1;
#pragma unroll
      for (int p = 0; p < NP; ++p) {   // row r = lane (< 8): its C sums sit in lane r >> 1, slot r & 1
        const int src = (lane >> 1) & 3;
        const float a0x = __shfl_sync(0xffffffffu, aC[2 * p].x, src), a0y = __shfl_sync(0xffffffffu, aC[2 * p].y, src);
        const float a1x = __shfl_sync(0xffffffffu, aC[2 * p + 1].x, src), a1y = __shfl_sync(0xffffffffu, aC[2 * p + 1].y, src);
        const float2 sum = make_float2(aW[p].x + ((lane & 1) ? a1x : a0x), aW[p].y + ((lane & 1) ? a1y : a0y));
        if (m >= 0) {
          if constexpr (PARTS) {
            float2* y = p ? y1 : y0;
            if (y) y[m] = p ? make_float2(-sum.x, -sum.y) : sum;
          } else {   // (j alpha) u: re = -alpha u.im, im = alpha u.re
            y0[m] = make_float2(-al * sum.y, al * sum.x);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 2 * NP; ++j) aC[j] = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < NP; ++j) aW[j] = make_float2(0.f, 0.f);
    }
    __syncwarp();   // every lane is done with stage k % NS: refill it
    if (lane == 0 && k + D < nch) issue(k + D, dn);
  }
}

// S4+S5 on the tensor cores (c64 batched launches, BB = 8/16/32 columns).
// The same chunk payload and TMA ring as k_interp_near; per row group the
// contraction is done as  D^T[2BB x 2R] += X^T[2BB x K] . C^T[K x 2R]  with
// mma.sync m16n8k8 tf32 (legacy tensor path, operands straight from the
// registers the gather loads into -- no shared-memory staging):
//   M = the 2BB real components of the batch (MT = BB/8 m16 tiles),
//   N = C chunks: two n8 tiles, the group's R = 8 rows of the A part (C^A)
//       and of the rho part (C^rho); W chunks: one n8 tile, the rho channel
//       entering A as -beta_b phi^rho (beta_b is a per-M-row scale), so the
//       tile accumulates Lambda^x,y,z . phi^x,y,z - beta_b Lambda^rho . phi^rho,
//   K = C chunk: the chunk's union entries (8 per k-step);
//       W chunk: (entry, channel) pairs (2 entries x 4 channels per k-step).
// fp32 accuracy by the 3-term split  a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi
// (a_hi = a truncated to tf32, a_lo = a - a_hi exact; the dropped a_lo b_lo
// and the truncation of a_lo, b_lo to tf32 are ~2^-20 relative).
// M mapping: lane (g = lane/4, t = lane%4) loads the 2MT contiguous reals
// q = 2MT g + 2j + h of its gathered rows (one or two 16-byte loads); tile j's
// fragment row g is q with h = 0 (the real part of column MT g + j), row
// g + 8 is h = 1 (its imaginary part).  The accumulator fragment then holds,
// for column b = MT g + j and rows r = 2t, 2t + 1, both parts (n tiles 0, 1)
// re and im in one lane, so the combine y = j alpha_b (y^A - beta_b y^rho)
// (eq:EFIEAIMx P:288) needs no shuffles; the four warps' partial sums are
// added in a fixed order through shared memory at the group's last chunk.
template <int MT> struct NearMma {
  static constexpr int NT = 128, R = 8, BB = 8 * MT;
  static constexpr int CHC = 128, CHW = 32;                 // largest chunk lengths (entries) at c64
  static constexpr int D = kNearD, NDS = D + 1, NDD = D + 1;
  static constexpr int STB = CHC * R * 8 + CHC * 4 + 16;    // stage: one chunk payload
  static constexpr int KB = 2;                              // k-steps per warp batch (loads in flight)
  static constexpr size_t OFF_RED = (size_t)NDS * STB;
  static constexpr size_t REDB = (size_t)4 * 32 * (4 * MT + 1) * sizeof(float);   // [warp][lane][2 rows][MT][re, im]
  static constexpr size_t OFF_DESC = (OFF_RED + REDB + 15) / 16 * 16;
  static constexpr size_t OFF_BAR = OFF_DESC + NDD * 16;
  static constexpr size_t OFF_NBE = OFF_BAR + NDS * 8;      // [BB] -beta_b
  static constexpr size_t SMEM = OFF_NBE + BB * 4;
};

// a -> (hi, lo) with hi + lo = a exactly, hi a tf32 (truncated: one LOP3;
// cvt.rna.tf32.f32 expands to five instructions on sm_100a), |lo| < 2^-10 |a|
__device__ __forceinline__ void tf32_split(float a, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(a) & 0xffffe000u;
  lo = __float_as_uint(a - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// the lane's 2MT contiguous reals of a gathered row (zero when !ok)
template <int MT> struct RowV { float v[2 * MT]; };
template <int MT>
__device__ __forceinline__ RowV<MT> load_row(const float* p, bool ok) {
  RowV<MT> r;
  if constexpr (MT == 4) {
    float4 u0 = make_float4(0.f, 0.f, 0.f, 0.f), u1 = u0;
    if (ok) { u0 = __ldg((const float4*)p); u1 = __ldg((const float4*)p + 1); }
    r.v[0] = u0.x; r.v[1] = u0.y; r.v[2] = u0.z; r.v[3] = u0.w;
    r.v[4] = u1.x; r.v[5] = u1.y; r.v[6] = u1.z; r.v[7] = u1.w;
  } else if constexpr (MT == 2) {
    float4 u0 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ok) u0 = __ldg((const float4*)p);
    r.v[0] = u0.x; r.v[1] = u0.y; r.v[2] = u0.z; r.v[3] = u0.w;
  } else {
    float2 u0 = make_float2(0.f, 0.f);
    if (ok) u0 = __ldg((const float2*)p);
    r.v[0] = u0.x; r.v[1] = u0.y;
  }
  return r;
}

template <int MT>
__global__ void __launch_bounds__(128, 5) k_interp_near_mma(HotDev h, const float2* __restrict__ xt, float2* __restrict__ y0,
                                                           Combine cb) {
  pdl_wait();
  pdl_trigger();
  using K = NearMma<MT>;
  constexpr int R = K::R, BB = K::BB, KB = K::KB;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* const sdata = smem;
  float* const red = reinterpret_cast<float*>(smem + K::OFF_RED);
  int4* const sdesc = reinterpret_cast<int4*>(smem + K::OFF_DESC);
  uint64_t* const bar = reinterpret_cast<uint64_t*>(smem + K::OFF_BAR);
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int c0 = h.cta_ptr[blockIdx.x], nch = h.cta_ptr[blockIdx.x + 1] - c0;
  if (nch <= 0) return;
  const int4* __restrict__ chunks = reinterpret_cast<const int4*>(h.chunks) + c0;
  const int nc = h.nc;
  const int64_t ns = (int64_t)h.batch * nc;                       // phi node stride (complex)
  const float* __restrict__ xr = reinterpret_cast<const float*>(xt) + 2 * MT * g;
  const float* __restrict__ phr = reinterpret_cast<const float*>(h.phi) + 2 * MT * g;
  // W chunks: this lane's channel t (x, y, z, rho) -> stored channel, or none
  // (planar grids store x, y, rho: Lambda^z = 0 and phi^z is not kept)
  const int wch = (nc == 3) ? (t == 3 ? 2 : (t == 2 ? -1 : t)) : t;
  float* const nbe = reinterpret_cast<float*>(smem + K::OFF_NBE) + MT * g;   // -beta of the lane's columns MT g + j
  if (tid < BB) reinterpret_cast<float*>(smem + K::OFF_NBE)[tid] = -(float)cb.beta[tid];
  float acc[MT][2][4];
#pragma unroll
  for (int j = 0; j < MT; ++j)
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[j][p][i] = 0.f;

  auto coef_bytes = [&](const int4& d) -> int { return d.w * R * ((d.y & 1) ? 8 : 16); };
  auto issue = [&](int j, const int4& d) {
    uint64_t* bj = bar + j % K::NDS;
    const uint32_t bytes = (uint32_t)(coef_bytes(d) + ((4 * d.w + 15) & ~15) + 16);
    sdesc[j % K::NDD] = d;
    mbar_arrive_expect_tx(bj, bytes);
    bulk_g2s(sdata + (j % K::NDS) * K::STB, h.payload + (int64_t)d.z * 16, bytes, bj);
  };
  if (tid < K::NDS) mbar_init(bar + tid, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  if (tid == 0)
    for (int j = 0; j < K::D && j < nch; ++j) issue(j, chunks[j]);
  __syncthreads();

  for (int k = 0; k < nch; ++k) {
    mbar_wait(bar + k % K::NDS, (uint32_t)(k / K::NDS) & 1u);
    const int4 d = sdesc[k % K::NDD];
    const unsigned char* stg = sdata + (k % K::NDS) * K::STB;
    const int* ix = reinterpret_cast<const int*>(stg + coef_bytes(d));
    if (tid == 0 && k + K::D < nch)
      issue(k + K::D, *reinterpret_cast<const int4*>(stg + coef_bytes(d) + ((4 * d.w + 15) & ~15)));
    const bool isC = d.y & 1;
    const int nks = isC ? (d.w + 7) >> 3 : (d.w + 1) >> 1, elast = d.w - 1;   // k-steps: 8 / 2 entries
    for (int ks0 = wib; ks0 < nks; ks0 += 4 * KB) {
      // gathered rows of KB k-steps, all loads before any use (k = t and t + 4).
      // Entries past the chunk load a valid row (the last entry's) against a
      // zero coefficient, so no load is predicated.
      RowV<MT> ra[KB][2];
      float bA[KB][2], bR[KB][2];
      if (isC) {
#pragma unroll
        for (int q = 0; q < KB; ++q)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int e = (ks0 + 4 * q) * 8 + t + 4 * hh;
            const int ec = min(e, elast);
            ra[q][hh] = load_row<MT>(xr + (int64_t)ix[ec] * (2 * BB), true);
            const float2 cv = reinterpret_cast<const float2*>(stg)[ec * R + g];
            bA[q][hh] = e <= elast ? cv.x : 0.f;
            bR[q][hh] = e <= elast ? cv.y : 0.f;
          }
      } else {
#pragma unroll
        for (int q = 0; q < KB; ++q)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int e = (ks0 + 4 * q) * 2 + hh;
            const int ec = min(e, elast);
            // planar grids: the absent z channel (t = 2) reads channel 0 against
            // a zero weight
            ra[q][hh] = load_row<MT>(phr + ((int64_t)ix[ec] * ns + (int64_t)max(wch, 0) * h.batch) * 2, true);
            // the rho channel enters as -beta_b phi^rho (beta_b scales M rows), so
            // one n tile carries y^A - beta y^rho of the W part
            if (t == 3)
#pragma unroll
              for (int j = 0; j < MT; ++j) {
                ra[q][hh].v[2 * j] *= nbe[j];
                ra[q][hh].v[2 * j + 1] *= nbe[j];
              }
            const float w = reinterpret_cast<const float*>(stg)[(ec * R + g) * 4 + t];
            bA[q][hh] = (e <= elast && wch >= 0) ? w : 0.f;
          }
      }
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        if (ks0 + 4 * q >= nks) break;   // warp-uniform
        uint32_t bh[2][2], bl[2][2];   // [part][k half]
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          tf32_split(bA[q][hh], bh[0][hh], bl[0][hh]);
          if (isC) tf32_split(bR[q][hh], bh[1][hh], bl[1][hh]);
        }
#pragma unroll
        for (int j = 0; j < MT; ++j) {
          uint32_t ah[4], al[4];
          tf32_split(ra[q][0].v[2 * j], ah[0], al[0]);       // (row g,     k = t)
          tf32_split(ra[q][0].v[2 * j + 1], ah[1], al[1]);   // (row g + 8, k = t)
          tf32_split(ra[q][1].v[2 * j], ah[2], al[2]);       // (row g,     k = t + 4)
          tf32_split(ra[q][1].v[2 * j + 1], ah[3], al[3]);   // (row g + 8, k = t + 4)
          mma_tf32(acc[j][0], al, bh[0][0], bh[0][1]);
          mma_tf32(acc[j][0], ah, bl[0][0], bl[0][1]);
          mma_tf32(acc[j][0], ah, bh[0][0], bh[0][1]);
          if (isC) {   // W chunks: one n tile (rho folded into A)
            mma_tf32(acc[j][1], al, bh[1][0], bh[1][1]);
            mma_tf32(acc[j][1], ah, bl[1][0], bl[1][1]);
            mma_tf32(acc[j][1], ah, bh[1][0], bh[1][1]);
          }
        }
      }
    }
    if (d.y & 4) {   // last chunk of group d.x: combine, fixed-order reduction over the warps, store
      // lane's outputs: column b = MT g + j, row r = 2t + hh; y^A - beta_b y^rho
      float* rw = red + (wib * 32 + lane) * (4 * MT + 1);
#pragma unroll
      for (int j = 0; j < MT; ++j) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          rw[(hh * MT + j) * 2] = acc[j][0][hh] + nbe[j] * acc[j][1][hh];             // re (fragment row g)
          rw[(hh * MT + j) * 2 + 1] = acc[j][0][2 + hh] + nbe[j] * acc[j][1][2 + hh];   // im (fragment row g + 8)
        }
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[j][p][i] = 0.f;
      }
      __syncthreads();
      const int32_t* gr = h.grp_rows + (int64_t)d.x * R;
      // 32 lanes x 2 rows x MT columns complex outputs
      for (int o = tid; o < 32 * 2 * MT; o += K::NT) {
        const int ln = o / (2 * MT), jj = o % (2 * MT);   // jj = hh MT + j
        float re = 0.f, im = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float* src = red + (w * 32 + ln) * (4 * MT + 1) + 2 * jj;
          re += src[0];
          im += src[1];
        }
        const int hh = jj / MT, j = jj % MT;
        const int b = MT * (ln >> 2) + j, r = 2 * (ln & 3) + hh;
        const int m = gr[r];
        if (m >= 0 && b < cb.B) {   // (j alpha) u: re = -alpha u.im, im = alpha u.re
          const float al = (float)cb.alpha_im[b];
          y0[(int64_t)b * cb.ystride + m] = make_float2(-al * im, al * re);
        }
      }
    }
    __syncthreads();   // stage, descriptor and reduction slots are reused next
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
    case 4: launch_pdl(k_gather<T, 4>, dim3(g), dim3(256), 0, s, h, (const T2*)x, xstride); break;
    case 8: launch_pdl(k_gather<T, 8>, dim3(g), dim3(256), 0, s, h, (const T2*)x, xstride); break;
    case 16: launch_pdl(k_gather<T, 16>, dim3(g), dim3(256), 0, s, h, (const T2*)x, xstride); break;
    default: launch_pdl(k_gather<T, 32>, dim3(g), dim3(256), 0, s, h, (const T2*)x, xstride); break;
  }
  AIMX_CHECK_LAUNCH();
}

template <typename T, int L, bool SMALL>
void run_x_geom(const HotDev& h, bool inv, int B, cudaStream_t s) {
  constexpr size_t sm = pass_smem<T, L, SMALL>();
  constexpr int NL = PassGeom<T, L, SMALL>::NL;
  dim3 g((unsigned)(((int64_t)h.nlines * h.nc + NL - 1) / NL), (unsigned)B);
  if (!inv) {
    set_smem(k_xfwd<T, L, SMALL>, sm);
    launch_pdl(k_xfwd<T, L, SMALL>, g, dim3(PassGeom<T, L, SMALL>::NT), sm, s, h);
  } else {
    set_smem(k_xinv<T, L, SMALL>, sm);
    launch_pdl(k_xinv<T, L, SMALL>, g, dim3(PassGeom<T, L, SMALL>::NT), sm, s, h);
  }
  AIMX_CHECK_LAUNCH();
}
template <typename T, int L, int NCH>
void run_x_b(const HotDev& h, int B, cudaStream_t s) {
  using X = XinvB<T, L, NCH>;
  set_smem(k_xinv_b<T, L, NCH>, X::SMEM);
  launch_pdl(k_xinv_b<T, L, NCH>, dim3((unsigned)h.nlines, (unsigned)((B + 3) / 4)), dim3(X::NT), X::SMEM, s, h, B);
  AIMX_CHECK_LAUNCH();
}

// x passes: below two waves of default CTAs, one x row per (smaller) CTA;
// batched inverse passes (B >= 4, lines of 64+ points) group 4 slots per CTA
template <typename T, int L>
void run_x(const HotDev& h, bool inv, int B, cudaStream_t s) {
  if (h.nlines <= 0) return;
  // batched inverse: 4 slots per CTA (the forward pass's per-slot CTAs already
  // read and write whole runs of channels; a batched forward measured slower:
  // cfg5 188 against 159 us)
  if (inv && B >= 4 && L >= 64 && h.batch % 4 == 0 && XinvB<T, L>::SMEM <= 220 * 1024) {
    if (h.nc == 3) run_x_b<T, L, 3>(h, B, s);
    else run_x_b<T, L, 4>(h, B, s);
    return;
  }
  constexpr int NL = PassGeom<T, L>::NL;
  if (((int64_t)h.nlines * h.nc + NL - 1) / NL * B < 2 * 148) run_x_geom<T, L, true>(h, inv, B, s);
  else run_x_geom<T, L, false>(h, inv, B, s);
}

template <typename T, int L> dim3 col_grid(int W, int rows, int B) {
  constexpr int NL = PassGeom<T, L>::NL;
  const int CW = col_width(W, NL);
  const int RPC = NL / CW;
  return dim3((unsigned)(W / CW), (unsigned)((rows + RPC - 1) / RPC), (unsigned)B);
}

template <typename T, int L>
void run_y(const HotDev& h, bool inv, int B, cudaStream_t s) {
  constexpr size_t sm = pass_smem<T, L>();
  dim3 g = col_grid<T, L>(h.W, h.nzocc, B);
  if (!inv) {
    set_smem(k_yfwd<T, L>, sm);
    launch_pdl(k_yfwd<T, L>, g, dim3(PassGeom<T, L>::NT), sm, s, h);
  } else {
    set_smem(k_yinv<T, L>, sm);
    launch_pdl(k_yinv<T, L>, g, dim3(PassGeom<T, L>::NT), sm, s, h);
  }
  AIMX_CHECK_LAUNCH();
}

// ---- z conv with ONE occupied z plane z0 (planar meshes, e.g. cfg5): the
// potentials are only needed on z0 (the inverse passes read occupied planes
// only), and for a single non-zero input the z forward * H_hat * z inverse at
// z0 collapses exactly to a multiply by the kernel's z-sum,
//   phi(z0) = v(z0) * sum_{kz < 2N_z} H_hat(kz) / M
//           = v(z0) * (H(0) + H(N_z) + 2 sum_{0 < kz < N_z} H(kz))   (octant, H even in kz).
// One thread per (ky, kx) and its 4 channel columns, in place on bufB.
template <typename T>
__global__ void k_zconv_plane(HotDev h) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  const int W = h.W, Nx = h.Nx, Ny = h.Ny, Nz = h.Nz, Ny2 = 2 * h.Ny, W4 = W / 4;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)Ny2 * W4) return;
  const int ky = (int)(i / W4), kxl = (int)(i - (int64_t)ky * W4);
  const int b = blockIdx.y;
  const int kx = h.kx0 + kxl;
  const int kxf = kx <= Nx ? kx : 2 * Nx - kx, kyf = ky <= Ny ? ky : Ny2 - ky;
  const T2* __restrict__ Hb = (const T2*)h.Hoct + b * h.sH + (int64_t)kyf * (Nz + 1) * (Nx + 1) + kxf;
  T2 f = Hb[0];
  T2 mid = mk<T2>(0, 0);
  for (int kz = 1; kz < Nz; ++kz) mid = cadd(mid, Hb[(int64_t)kz * (Nx + 1)]);
  const T2 last = Hb[(int64_t)Nz * (Nx + 1)];
  f.x += last.x + 2 * mid.x;
  f.y += last.y + 2 * mid.y;
  T2* __restrict__ g = (T2*)h.bufB + b * h.sB + (int64_t)h.zplane0 * Ny2 * W + (int64_t)ky * W + 4 * kxl;
#pragma unroll
  for (int c = 0; c < 4; ++c) g[c] = cmul(g[c], f);
}

template <typename T, int L>
void run_z(const HotDev& h, int B, cudaStream_t s) {
  if (h.nzocc == 1) {
    const int64_t n = (int64_t)2 * h.Ny * (h.W / 4);
    launch_pdl(k_zconv_plane<T>, dim3((unsigned)((n + 255) / 256), (unsigned)B), dim3(256), 0, s, h);
    AIMX_CHECK_LAUNCH();
    return;
  }
  // + two spectrum slabs: NL lines x L / 4 complex (RPC * L * CW / 4) each
  constexpr size_t sm = pass_smem<T, L>() + 2 * sizeof(typename CT<T>::T2) * (size_t)PassGeom<T, L>::NL * L / 4;
  dim3 g = col_grid<T, L>(h.W, 2 * h.Ny, B);
  g.y = (g.y + ZROWS - 1) / ZROWS;   // row sets per CTA
  if (h.tmB && h.nzocc == h.Nz && h.W >= ZGeom<T, L>::NL && h.W % ZGeom<T, L>::NL == 0 && h.Nz <= 256) {
    using Z = ZTma<T, L>;
    const size_t zs = Z::smem(h.Nz);
    set_smem(k_zconv_tma<T, L>, zs);
    dim3 gt((unsigned)(h.W / Z::CW), (unsigned)((2 * h.Ny + ZROWS - 1) / ZROWS), (unsigned)B);
    launch_pdl(k_zconv_tma<T, L>, gt, dim3(ZGeom<T, L>::NT), zs, s, h, *(const CUtensorMap*)h.tmB);
  } else if (h.nzocc == h.Nz) {
    set_smem(k_zconv<T, L, true>, sm);
    launch_pdl(k_zconv<T, L, true>, g, dim3(PassGeom<T, L>::NT), sm, s, h);
  } else {
    set_smem(k_zconv<T, L, false>, sm);
    launch_pdl(k_zconv<T, L, false>, g, dim3(PassGeom<T, L>::NT), sm, s, h);
  }
  AIMX_CHECK_LAUNCH();
}

// xt[n * BB + b] = x[b * xstride + n] (zero for b >= B): a transpose through a
// shared-memory tile of kIlN rows, so both the column reads (kIlN consecutive
// n of a column) and the interleaved writes (kIlN * BB contiguous) coalesce
constexpr int kIlN = 64;
template <typename T>
__global__ void __launch_bounds__(256) k_interleave(int nb, int B, int BB, const typename CT<T>::T2* __restrict__ x,
                                                    int64_t xstride, typename CT<T>::T2* __restrict__ xt) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  __shared__ T2 tile[kMaxBatch][kIlN + 1];
  const int n0 = blockIdx.x * kIlN;
  for (int idx = threadIdx.x; idx < BB * kIlN; idx += blockDim.x) {
    const int b = idx / kIlN, j = idx - b * kIlN;
    tile[b][j] = (b < B && n0 + j < nb) ? x[b * xstride + n0 + j] : mk<T2>(0, 0);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < BB * kIlN; idx += blockDim.x) {
    const int j = idx / BB, b = idx - j * BB;
    if (n0 + j < nb) xt[(int64_t)(n0 + j) * BB + b] = tile[b][j];
  }
}

template <int BB> constexpr int bucket_ok() { return BB; }
inline int batch_bucket(int B) { return B <= 1 ? 1 : (B <= 2 ? 2 : (B <= 4 ? 4 : (B <= 8 ? 8 : (B <= 16 ? 16 : 32)))); }

template <typename T>
void run_interleave(const HotDev& h, const void* x, const Combine& c, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const int BB = batch_bucket(c.B);
  launch_pdl(k_interleave<T>, dim3((unsigned)((h.nb + kIlN - 1) / kIlN)), dim3(256), 0, s, h.nb, c.B, BB, (const T2*)x,
             c.xstride, (T2*)h.xt);
  AIMX_CHECK_LAUNCH();
}

template <typename T>
void run_gather_b(const HotDev& h, int B, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const unsigned g = (unsigned)(((int64_t)h.nocc * 32 + 255) / 256);
  const T2* xt = (const T2*)h.xt;
  switch (batch_bucket(B)) {
    case 2: launch_pdl(k_gather_b<T, 2>, dim3(g), dim3(256), 0, s, h, xt, B); break;
    case 4: launch_pdl(k_gather_b<T, 4>, dim3(g), dim3(256), 0, s, h, xt, B); break;
    case 8: launch_pdl(k_gather_b<T, 8>, dim3(g), dim3(256), 0, s, h, xt, B); break;
    case 16: launch_pdl(k_gather_b<T, 16>, dim3(g), dim3(256), 0, s, h, xt, B); break;
    default: launch_pdl(k_gather_b<T, 32>, dim3(g), dim3(256), 0, s, h, xt, B); break;
  }
  AIMX_CHECK_LAUNCH();
}

template <typename T, int R, int BB, bool PARTS>
void launch_interp(const HotDev& h, const void* xt, void* y0, void* y1, const Combine& c, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  using K = NearCfg<T, R, BB, PARTS>;
  set_smem(k_interp_near<T, R, BB, PARTS>, K::SMEM);
  launch_pdl(k_interp_near<T, R, BB, PARTS>, dim3((unsigned)(BB == 1 ? h.near_ctas1 : h.near_ctas)), dim3(K::NT), K::SMEM, s, h, (const T2*)xt, (T2*)y0,
                                                                                 (T2*)y1, c);
  AIMX_CHECK_LAUNCH();
}

template <int MT>
void launch_interp_mma(const HotDev& h, void* y0, const Combine& c, cudaStream_t s) {
  using K = NearMma<MT>;
  set_smem(k_interp_near_mma<MT>, K::SMEM);
  launch_pdl(k_interp_near_mma<MT>, dim3((unsigned)h.near_ctas), dim3(K::NT), K::SMEM, s, h, (const float2*)h.xt,
             (float2*)y0, c);
  AIMX_CHECK_LAUNCH();
}

template <typename T, int R>
void run_interp_r(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s) {
  (void)x;
  if (c.B == 1) {   // single column, staged in xt by run_interleave
    if constexpr (sizeof(T) == 4 && R == 8) {   // c64: rows split over lanes
      if (!h.near1_old) {
        auto go = [&](auto kern, size_t smem) {
          set_smem(kern, smem);
          launch_pdl(kern, dim3((unsigned)h.near_ctas1), dim3(128), smem, s, h, (const float2*)h.xt, (float2*)y0,
                     (float2*)y1, c);
        };
        if (h.near_half && h.warp_ptr1) {   // warp-private rings (32-slot contexts)
          auto gow = [&](auto kern) {
            set_smem(kern, Near1W::SMEM);
            launch_pdl(kern, dim3((unsigned)(h.near_warps1 / Near1W::NW)), dim3(Near1W::NT), Near1W::SMEM, s, h,
                       (const float2*)h.xt, (float2*)y0, (float2*)y1, c);
          };
          if (c.mode == 1) gow(k_interp_near1w<true>);
          else gow(k_interp_near1w<false>);
          AIMX_CHECK_LAUNCH();
          return;
        }
        if (h.near_half) {   // near_chc / near_chw of this context's payload
          if (c.mode == 1) go(k_interp_near1<true, true>, Near1Smem<true, true>::SMEM);
          else go(k_interp_near1<false, true>, Near1Smem<false, true>::SMEM);
        } else {
          if (c.mode == 1) go(k_interp_near1<true, false>, Near1Smem<true, false>::SMEM);
          else go(k_interp_near1<false, false>, Near1Smem<false, false>::SMEM);
        }
        AIMX_CHECK_LAUNCH();
        return;
      }
    }
    if (c.mode == 1) launch_interp<T, R, 1, true>(h, h.xt, y0, y1, c, s);
    else launch_interp<T, R, 1, false>(h, h.xt, y0, y1, c, s);
    return;
  }
  if (c.mode != 0) throw Error(AIMX_E_INTERNAL, "batched parts not supported");
  if constexpr (sizeof(T) == 4 && R == 8) {   // c64, 8 to 32 columns: the tensor-core kernel (opt-in)
    // opt-in (AIMX_NEAR_MMA=1 at setup): measured slower than the FMA kernel on
    // B200 (legacy HMMA issue rate, 3-term split)
    const int bb = batch_bucket(c.B);
    if (h.near_mma && bb >= 8) {
      switch (bb) {
        case 8: launch_interp_mma<1>(h, y0, c, s); break;
        case 16: launch_interp_mma<2>(h, y0, c, s); break;
        default: launch_interp_mma<4>(h, y0, c, s); break;
      }
      return;
    }
  }
  switch (batch_bucket(c.B)) {   // xt: interleaved by run_interleave earlier in the matvec
    case 2: launch_interp<T, R, 2, false>(h, h.xt, y0, y1, c, s); break;
    case 4: launch_interp<T, R, 4, false>(h, h.xt, y0, y1, c, s); break;
    case 8: launch_interp<T, R, 8, false>(h, h.xt, y0, y1, c, s); break;
    case 16: launch_interp<T, R, 16, false>(h, h.xt, y0, y1, c, s); break;
    default: launch_interp<T, R, 32, false>(h, h.xt, y0, y1, c, s); break;
  }
}

// Linear-term modification: y^A += k0^2 C^A_lin x, y^rho += k0^2
// C^rho_lin x over the <= kLinW overlapping columns of each row, after S4+S5
// (combined: y += j alpha (k0^2 C^A_lin x - C^rho_lin x); PARTS: y0 += k0^2
// C^A_lin x, y1 -= k0^2 C^rho_lin x).  Thread per (row, column of the batch):
// the batch-interleaved xt makes the x reads of a row's threads contiguous.
template <typename T, bool PARTS>
__global__ void k_lin(const int32_t* __restrict__ lcol, const typename CT<T>::T2* __restrict__ lc, int nb, int BB,
                      const typename CT<T>::T2* __restrict__ xt, typename CT<T>::T2* __restrict__ y0,
                      typename CT<T>::T2* __restrict__ y1, Combine cb) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)nb * BB) return;
  const int m = (int)(i / BB), b = (int)(i - (int64_t)m * BB);
  if (b >= cb.B) return;
  T2 sa = mk<T2>(0, 0), sr = mk<T2>(0, 0);
#pragma unroll
  for (int j = 0; j < kLinW; ++j) {
    const int n = lcol[m * kLinW + j];
    if (n < 0) continue;
    const T2 c = lc[m * kLinW + j];
    const T2 xv = xt[(int64_t)n * BB + b];
    sa.x += c.x * xv.x; sa.y += c.x * xv.y;
    sr.x += c.y * xv.x; sr.y += c.y * xv.y;
  }
  const T k2 = (T)(1.0 / cb.beta[b]);
  if constexpr (PARTS) {
    if (y0) { T2 v = y0[m]; v.x += k2 * sa.x; v.y += k2 * sa.y; y0[m] = v; }
    if (y1) { T2 v = y1[m]; v.x -= k2 * sr.x; v.y -= k2 * sr.y; y1[m] = v; }
  } else {
    const T al = (T)cb.alpha_im[b];
    const T ux = k2 * sa.x - sr.x, uy = k2 * sa.y - sr.y;
    T2* y = y0 + (int64_t)b * cb.ystride + m;
    T2 v = *y;
    v.x -= al * uy;
    v.y += al * ux;
    *y = v;
  }
}

template <typename T>
void run_lin(const HotDev& h, void* y0, void* y1, const Combine& c, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const int BB = batch_bucket(c.B);
  const int64_t n = (int64_t)h.nb * BB;
  const unsigned g = (unsigned)((n + 255) / 256);
  if (c.mode == 1)
    launch_pdl(k_lin<T, true>, dim3(g), dim3(256), 0, s, (const int32_t*)h.lin_col, (const T2*)h.lin_c, h.nb, BB,
               (const T2*)h.xt, (T2*)y0, (T2*)y1, c);
  else
    launch_pdl(k_lin<T, false>, dim3(g), dim3(256), 0, s, (const int32_t*)h.lin_col, (const T2*)h.lin_c, h.nb, BB,
               (const T2*)h.xt, (T2*)y0, (T2*)y1, c);
  AIMX_CHECK_LAUNCH();
}

template <typename T>
void run_interp(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s) {
  if (h.R == 4) run_interp_r<T, 4>(h, x, y0, y1, c, s);
  else if (h.R == 16) run_interp_r<T, 16>(h, x, y0, y1, c, s);
  else run_interp_r<T, 8>(h, x, y0, y1, c, s);
}

template <typename T, int L> void run_yconv_plane(const HotDev& h, int B, cudaStream_t s) {
  // the slab: kx of the tile's columns (CW/3 + 2 at most), + the occupied-row flags
  constexpr size_t sm = pass_smem<T, L>() + sizeof(typename CT<T>::T2) * (size_t)(L / 2 + 1) * (PassGeom<T, L>::NL / 3 + 2)
                        + L / 2;
  set_smem(k_yconv_plane<T, L>, sm);
  launch_pdl(k_yconv_plane<T, L>, col_grid<T, L>(h.W, 1, B), dim3(PassGeom<T, L>::NT), sm, s, h);
  AIMX_CHECK_LAUNCH();
}

// y fwd + z conv + y inv in one kernel when both transforms are short
// (reported as stage 3, zconv); CURL: the double-layer operator's spectral
// cross product (three gradient spectra) in place of the multiply
template <typename T, int LY, int LZ, bool CURL = false> void launch_yz(const HotDev& h, int B, cudaStream_t s) {
  using G = YZGeom<T, LY, LZ>;
  set_smem(k_yzconv<T, LY, LZ, CURL>, G::SMEM);
  dim3 g((unsigned)(h.W / G::TW), (unsigned)B);
  launch_pdl(k_yzconv<T, LY, LZ, CURL>, dim3(g), dim3(G::NT), G::SMEM, s, h);
  AIMX_CHECK_LAUNCH();
}
// CURL keeps three z lines per thread in registers: short z transforms only
template <typename T> constexpr int curl_fused_max_lz() { return sizeof(T) == 4 ? 16 : 8; }
template <typename T, bool CURL = false> bool run_yz_fused(const HotDev& h, int B, cudaStream_t s, Profiler* prof) {
  const int Ly = 2 * h.Ny, Lz = 2 * h.Nz;
  if (Ly > 32 || Lz > 32 || h.W % YZGeom<T, 8, 8>::TW != 0 || Ly * Lz > 512) return false;
  if (CURL && Lz > curl_fused_max_lz<T>()) return false;
  StageScope sc(prof, 3, s);
  switch (Ly * 64 + Lz) {
    case 8 * 64 + 8: launch_yz<T, 8, 8, CURL>(h, B, s); break;
    case 16 * 64 + 8: launch_yz<T, 16, 8, CURL>(h, B, s); break;
    case 32 * 64 + 8: launch_yz<T, 32, 8, CURL>(h, B, s); break;
    case 8 * 64 + 16: if constexpr (!CURL || curl_fused_max_lz<T>() >= 16) launch_yz<T, 8, 16, CURL>(h, B, s); break;
    case 16 * 64 + 16: if constexpr (!CURL || curl_fused_max_lz<T>() >= 16) launch_yz<T, 16, 16, CURL>(h, B, s); break;
    case 32 * 64 + 16: if constexpr (!CURL || curl_fused_max_lz<T>() >= 16) launch_yz<T, 32, 16, CURL>(h, B, s); break;
    case 8 * 64 + 32: if constexpr (!CURL) launch_yz<T, 8, 32>(h, B, s); break;
    case 16 * 64 + 32: if constexpr (!CURL) launch_yz<T, 16, 32>(h, B, s); break;
    default: return false;
  }
  return true;
}

// the z pass of the double-layer operator: TMA z pass with the spectral cross product
template <typename T, int L> void run_z_curl(const HotDev& h, cudaStream_t s) {
  using Z = ZTma<T, L, true>;
  const size_t zs = Z::smem(h.Nz);
  set_smem(k_zconv_tma<T, L, true>, zs);
  dim3 gt((unsigned)(h.W / Z::CW), (unsigned)((2 * h.Ny + ZROWS - 1) / ZROWS), 1u);
  launch_pdl(k_zconv_tma<T, L, true>, gt, dim3(ZGeom<T, L>::NT), zs, s, h, *(const CUtensorMap*)h.tmB);
  AIMX_CHECK_LAUNCH();
}
template <typename T> bool z_curl_tma_ok(const HotDev& h) {
  int nl = 0;
  AIMX_SWITCH_L(2 * h.Nz, (nl = ZGeom<T, L>::NL));
  return h.tmB && h.nzocc == h.Nz && h.W >= nl && h.W % nl == 0 && h.Nz <= 256;
}

// S3 between the x transforms: the planar y pass, the fused short y/z pass,
// or y fwd / z conv / y inv (reported as stages 2, 3, 4; fused forms as 3)
template <typename T>
void grid_conv(const HotDev& h, int B, cudaStream_t s, Profiler* prof) {
  const int Ly = 2 * h.Ny, Lz = 2 * h.Nz;
  if (h.planar) {
    StageScope sc(prof, 3, s);
    AIMX_SWITCH_L(Ly, (run_yconv_plane<T, L>(h, B, s)));
    return;
  }
  if (run_yz_fused<T>(h, B, s, prof)) return;
  { StageScope sc(prof, 2, s); AIMX_SWITCH_L(Ly, (run_y<T, L>(h, false, B, s))); }
  { StageScope sc(prof, 3, s); AIMX_SWITCH_L(Lz, (run_z<T, L>(h, B, s))); }
  { StageScope sc(prof, 4, s); AIMX_SWITCH_L(Ly, (run_y<T, L>(h, true, B, s))); }
}

// S2 + S3 (+ x inverse): the grid part of a matvec, up to the potentials phi
template <typename T>
void hot_grid(const HotDev& h, const void* x, const Combine& c, cudaStream_t s, Profiler* prof) {
  if (c.B < 1 || c.B > h.batch || c.B > kMaxBatch) throw Error(AIMX_E_INTERNAL, "bad batch");
  const int Lx = 2 * h.Nx, B = c.B;
  {
    StageScope sc(prof, 1, s);
    if (!c.xt_ready) run_interleave<T>(h, x, c, s);   // xt: batch-interleaved columns (gather, S4+S5)
    if (B == 1) run_gather<T>(h, x, c.xstride, B, s);
    else run_gather_b<T>(h, B, s);
    AIMX_SWITCH_L(Lx, (run_x<T, L>(h, false, B, s)));
  }
  if (h.spec_ready) AIMX_CUDA(cudaStreamWaitEvent(s, h.spec_ready, 0));   // the batch's spectra
  grid_conv<T>(h, B, s, prof);
  { StageScope sc(prof, 5, s); AIMX_SWITCH_L(Lx, (run_x<T, L>(h, true, B, s))); }
}

// S4 + S5 (+ the linear-term correction): from phi and xt to y
template <typename T>
void hot_near(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s,
              Profiler* prof) {
  StageScope sc(prof, 6, s);
  run_interp<T>(h, x, y0, y1, c, s);
  if (h.lin_col) run_lin<T>(h, y0, y1, c, s);
}

template <typename T>
void hot_matvec(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s,
                Profiler* prof) {
  hot_grid<T>(h, x, c, s, prof);
  hot_near<T>(h, x, y0, y1, c, s, prof);
}

// ---- the double-layer operator K: its grid part
// through the EVEN radial factor F of grad G = -r F:
//   sum_{a,b} eps_cab (d_a G (*) J_b) = -h [s x (F (*) J) - F (*) (s x J)]_c,
// s the node coordinates in cells; two passes of the hot-path transforms with
// the spectrum F_hat, then y_K = -sum_c W^c Phi_c + C_K x.
// S := s x S on the occupied nodes (channel 3 -> 0), in place
template <typename T>
__global__ void k_cross_s(HotDev h) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= h.nocc) return;
  const int lin = h.node_lin[q];
  // coordinates about the grid centre (any origin is exact; the centre halves
  // |s| and with it the fp32 cancellation of s x (F * J) - F * (s x J))
  const T sx = (T)(lin % h.Nx - h.Nx / 2), sy = (T)((lin / h.Nx) % h.Ny - h.Ny / 2),
          sz = (T)(lin / (h.Nx * h.Ny) - h.Nz / 2);
  T2* g = (T2*)h.S + ((int64_t)h.node_line[q] * h.Nx + lin % h.Nx) * 4;
  const T2 jx = g[0], jy = g[1], jz = g[2];
  g[0] = mk<T2>(sy * jz.x - sz * jy.x, sy * jz.y - sz * jy.y);
  g[1] = mk<T2>(sz * jx.x - sx * jz.x, sz * jx.y - sx * jz.y);
  g[2] = mk<T2>(sx * jy.x - sy * jx.x, sx * jy.y - sy * jx.y);
  g[3] = mk<T2>(0, 0);
}

// warp per RWG: y = -sum_c sum_s Lambda^c[s] Phi_c(node), Phi = -hg [s x phi1 - phi2]
// (phi layout [node][channel][slot], slot 0; lanes over the stencil slots),
// then + C_K x (lanes over the row's CSR entries); fixed-order shuffle sum
template <typename T>
__global__ void k_kop_interp(HotDev h, const typename CT<T>::T2* __restrict__ phi1,
                             const typename CT<T>::T2* __restrict__ phi2, const double* __restrict__ lam,
                             double hg, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                             const T* __restrict__ ck, const typename CT<T>::T2* __restrict__ x,
                             typename CT<T>::T2* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  const int lane = threadIdx.x & 31;
  const int m = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (m >= h.nb) return;
  const int p = h.p, p3 = h.p3, Nx = h.Nx, Ny = h.Ny;
  const int64_t ns = (int64_t)h.batch * 4;
  const int base = h.rwg_base[m];
  double yr = 0.0, yi = 0.0;
  for (int sl = lane; sl < p3; sl += 32) {
    const double* lw = lam + ((int64_t)m * p3 + sl) * 4;
    if (lw[0] == 0.0 && lw[1] == 0.0 && lw[2] == 0.0) continue;
    const int i = sl % p, j = (sl / p) % p, k = sl / (p * p);
    const int lin = base + i + Nx * (j + Ny * k);
    const double s0 = lin % Nx - Nx / 2, s1 = (lin / Nx) % Ny - Ny / 2, s2 = lin / (Nx * Ny) - h.Nz / 2;
    const T2* a = phi1 + (int64_t)(lin - h.phi_off) * ns;
    const T2* b = phi2 + (int64_t)(lin - h.phi_off) * ns;
    const double ax = a[0].x, ay = a[h.batch].x, az = a[2 * h.batch].x;
    const double axi = a[0].y, ayi = a[h.batch].y, azi = a[2 * h.batch].y;
    const double px = -hg * ((s1 * az - s2 * ay) - b[0].x), pxi = -hg * ((s1 * azi - s2 * ayi) - b[0].y);
    const double py = -hg * ((s2 * ax - s0 * az) - b[h.batch].x), pyi = -hg * ((s2 * axi - s0 * azi) - b[h.batch].y);
    const double pz = -hg * ((s0 * ay - s1 * ax) - b[2 * h.batch].x), pzi = -hg * ((s0 * ayi - s1 * axi) - b[2 * h.batch].y);
    yr -= lw[0] * px + lw[1] * py + lw[2] * pz;
    yi -= lw[0] * pxi + lw[1] * pyi + lw[2] * pzi;
  }
  for (int64_t e = rowptr[m] + lane; e < rowptr[m + 1]; e += 32) {
    const T2 xv = x[col[e]];
    yr += (double)ck[e] * xv.x;
    yi += (double)ck[e] * xv.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    yr += __shfl_xor_sync(0xffffffffu, yr, o);
    yi += __shfl_xor_sync(0xffffffffu, yi, o);
  }
  if (lane == 0) y[m] = mk<T2>((T)yr, (T)yi);
}

template <typename T>
void hot_kop(const HotDev& h0, const void* x, void* y, const void* HF, void* phi1, void* phi2, const double* lam,
             double hg, const int64_t* rowptr, const int32_t* col, const void* ck, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  HotDev h = h0;
  h.Hoct = const_cast<void*>(HF);
  h.batch = 1;   // one column: compact potentials ([node][channel])
  if (h.nc != 4) {   // s x J has a z component on planar meshes: K keeps 4 channels, its own S
    h.nc = 4;
    h.W = 8 * h.Nx;
    h.S = h.S4;
  }
  const int Lx = 2 * h.Nx;
  run_gather<T>(h, x, h.nb, 1, s);   // S = P x (one column)
  auto conv = [&](void* phi) {
    h.phi = phi;
    AIMX_SWITCH_L(Lx, (run_x<T, L>(h, false, 1, s)));
    grid_conv<T>(h, 1, s, nullptr);
    AIMX_SWITCH_L(Lx, (run_x<T, L>(h, true, 1, s)));
  };
  conv(phi1);                                   // F (*) J
  if (h.nocc > 0) {
    launch_pdl(k_cross_s<T>, dim3((unsigned)((h.nocc + 255) / 256)), dim3(256), 0, s, h);
    AIMX_CHECK_LAUNCH();
  }
  conv(phi2);                                   // F (*) (s x J)
  launch_pdl(k_kop_interp<T>, dim3((unsigned)(((int64_t)h.nb * 32 + 255) / 256)), dim3(256), 0, s, h, (const T2*)phi1,
             (const T2*)phi2, lam, hg, rowptr, col, (const T*)ck, (const T2*)x, (T2*)y);
  AIMX_CHECK_LAUNCH();
}

// ---- the double-layer operator K through the gradient-of-kernel spectra
// (eq:KAIMx P:457, BASELINE cfg4 "K via gradient-of-kernel spectra"):
// Phi_c = sum_{a,b} eps_cab (d_a G (*) J_b) is ONE forward transform of the
// current channels, the spectral cross product Phi_hat = G_hat x J_hat with
// the three odd gradient spectra (octants, sign change past N_a along a) in
// the z pass, and ONE inverse transform; then y_K = -sum_c W^c Phi_c + C_K x.
// No cancellation: every term is the same size as the result, so c64 keeps
// its accuracy on flat faces (the radial form s x (F * J) - F * (s x J)
// cancels there).
template <typename T> bool kop_grad_ok(const HotDev& h) {
  if (h.planar) return false;
  const int Ly = 2 * h.Ny, Lz = 2 * h.Nz;
  const bool fused = Ly <= 32 && Lz <= curl_fused_max_lz<T>() && h.W % YZGeom<T, 8, 8>::TW == 0 &&
                     Ly * Lz <= 512 && Ly >= 8;
  return fused || z_curl_tma_ok<T>(h);
}

template <typename T>
void grid_conv_curl(const HotDev& h, cudaStream_t s) {
  if (run_yz_fused<T, true>(h, 1, s, nullptr)) return;
  const int Ly = 2 * h.Ny, Lz = 2 * h.Nz;
  AIMX_SWITCH_L(Ly, (run_y<T, L>(h, false, 1, s)));
  AIMX_SWITCH_L(Lz, (run_z_curl<T, L>(h, s)));
  AIMX_SWITCH_L(Ly, (run_y<T, L>(h, true, 1, s)));
}

// warp per RWG: y = -sum_{c in xyz} sum_s Lambda^c[s] Phi_c(node) + C_K x
// (phi: [node][channel], one column; fixed-order shuffle sum)
template <typename T>
__global__ void k_kop_interp_grad(HotDev h, const typename CT<T>::T2* __restrict__ phi,
                                  const double* __restrict__ lam, const int64_t* __restrict__ rowptr,
                                  const int32_t* __restrict__ col, const T* __restrict__ ck,
                                  const typename CT<T>::T2* __restrict__ x, typename CT<T>::T2* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  const int lane = threadIdx.x & 31;
  const int m = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (m >= h.nb) return;
  const int p = h.p, p3 = h.p3, Nx = h.Nx, Ny = h.Ny;
  const int base = h.rwg_base[m];
  double yr = 0.0, yi = 0.0;
  for (int sl = lane; sl < p3; sl += 32) {
    const double* lw = lam + ((int64_t)m * p3 + sl) * 4;
    if (lw[0] == 0.0 && lw[1] == 0.0 && lw[2] == 0.0) continue;
    const int i = sl % p, j = (sl / p) % p, k = sl / (p * p);
    const int64_t lin = base + i + Nx * (j + Ny * k);
    const T2* a = phi + (lin - h.phi_off) * 4;
    yr -= lw[0] * (double)a[0].x + lw[1] * (double)a[1].x + lw[2] * (double)a[2].x;
    yi -= lw[0] * (double)a[0].y + lw[1] * (double)a[1].y + lw[2] * (double)a[2].y;
  }
  for (int64_t e = rowptr[m] + lane; e < rowptr[m + 1]; e += 32) {
    const T2 xv = x[col[e]];
    yr += (double)ck[e] * xv.x;
    yi += (double)ck[e] * xv.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    yr += __shfl_xor_sync(0xffffffffu, yr, o);
    yi += __shfl_xor_sync(0xffffffffu, yi, o);
  }
  if (lane == 0) y[m] = mk<T2>((T)yr, (T)yi);
}

template <typename T>
void hot_kop_grad(const HotDev& h0, const void* x, void* y, const void* HG, void* phi, const double* lam,
                  const int64_t* rowptr, const int32_t* col, const void* ck, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  HotDev h = h0;
  h.Hoct = const_cast<void*>(HG);   // [3][noct]: d_x G, d_y G, d_z G
  h.batch = 1;                      // one column: compact potentials ([node][channel])
  h.phi = phi;
  const int Lx = 2 * h.Nx;
  run_gather<T>(h, x, h.nb, 1, s);                 // J = P x (the rho channel is carried, unused)
  AIMX_SWITCH_L(Lx, (run_x<T, L>(h, false, 1, s)));
  grid_conv_curl<T>(h, s);
  AIMX_SWITCH_L(Lx, (run_x<T, L>(h, true, 1, s)));
  launch_pdl(k_kop_interp_grad<T>, dim3((unsigned)(((int64_t)h.nb * 32 + 255) / 256)), dim3(256), 0, s, h,
             (const T2*)phi, lam, rowptr, col, (const T*)ck, (const T2*)x, (T2*)y);
  AIMX_CHECK_LAUNCH();
}

// ---- slab-decomposed hot path (SlabRank): per rank S2 + x fwd on its rows,
// exchange 0 (rows -> kx slabs), y fwd / z conv / y inv on its kx slab,
// exchange 1 (kx slabs -> rows incl. the `order`-row halo), x inv of its
// rows, S4 + S5 for its testing functions.
template <typename T>
void slab_matvec_t(std::vector<SlabRank*>& ranks, int Nx, int Ny, int Nz, SlabExchange& xchg, const void* x,
                   void* y0, void* y1, const Combine& c, cudaStream_t s, Profiler* prof) {
  if (c.B < 1 || c.B > kMaxBatch) throw Error(AIMX_E_INTERNAL, "bad batch");
  const int Lx = 2 * Nx, Ly = 2 * Ny, Lz = 2 * Nz, B = c.B;
  using T2 = typename CT<T>::T2;
  {
    StageScope sc(prof, 1, s);
    for (SlabRank* r : ranks) {
      run_interleave<T>(r->hr, x, c, s);
      if (r->hr.nocc > 0) {   // a rank's rows may hold no occupied node
        if (B == 1) run_gather<T>(r->hr, x, c.xstride, B, s);
        else run_gather_b<T>(r->hr, B, s);
      }
      if (r->hr.nlines > 0) AIMX_SWITCH_L(Lx, (run_x<T, L>(r->hr, false, B, s)));
    }
    xchg.run(ranks, 0, B, sizeof(T2), s);
  }
  for (SlabRank* r : ranks) {
    const HotDev& h = r->hc;
    if (!run_yz_fused<T>(h, B, s, prof)) {
      { StageScope sc(prof, 2, s); AIMX_SWITCH_L(Ly, (run_y<T, L>(h, false, B, s))); }
      { StageScope sc(prof, 3, s); AIMX_SWITCH_L(Lz, (run_z<T, L>(h, B, s))); }
      { StageScope sc(prof, 4, s); AIMX_SWITCH_L(Ly, (run_y<T, L>(h, true, B, s))); }
    }
  }
  {
    StageScope sc(prof, 5, s);
    xchg.run(ranks, 1, B, sizeof(T2), s);
    for (SlabRank* r : ranks)
      if (r->hx.nlines > 0) AIMX_SWITCH_L(Lx, (run_x<T, L>(r->hx, true, B, s)));
  }
  {
    StageScope sc(prof, 6, s);
    for (SlabRank* r : ranks)
      if (r->hr.ngrp > 0) {
        run_interp<T>(r->hr, x, y0, y1, c, s);
        if (r->hr.lin_col) run_lin<T>(r->hr, y0, y1, c, s);
      }
  }
}

// dst[i0][i1][i2][i3] = src[i0][i1][i2][i3] with per-axis strides (complex units)
template <typename T2>
__global__ void k_copy4(T2* __restrict__ dst, int64_t t0, int64_t t1, int64_t t2, const T2* __restrict__ src,
                        int64_t s0, int64_t s1, int64_t s2, int64_t d1, int64_t d2, int64_t d3, int64_t n) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t i3 = i % d3;
  int64_t r = i / d3;
  const int64_t i2 = r % d2;
  r /= d2;
  const int64_t i1 = r % d1, i0 = r / d1;
  dst[i0 * t0 + i1 * t1 + i2 * t2 + i3] = src[i0 * s0 + i1 * s1 + i2 * s2 + i3];
}

}  // namespace

void slab_matvec(std::vector<SlabRank*>& ranks, int Ny, int Nz, int Nx, bool f32, SlabExchange& xchg,
                 const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s, Profiler* prof) {
  if (f32) slab_matvec_t<float>(ranks, Nx, Ny, Nz, xchg, x, y0, y1, c, s, prof);
  else slab_matvec_t<double>(ranks, Nx, Ny, Nz, xchg, x, y0, y1, c, s, prof);
}

void copy4(void* dst, const int64_t t[3], const void* src, const int64_t st[3], const int64_t d[4], size_t csize,
           cudaStream_t s) {
  const int64_t n = d[0] * d[1] * d[2] * d[3];
  if (n <= 0) return;
  const unsigned g = (unsigned)((n + 255) / 256);
  if (csize == 8)
    launch_pdl(k_copy4<float2>, dim3(g), dim3(256), 0, s, (float2*)dst, t[0], t[1], t[2], (const float2*)src, st[0], st[1], st[2], d[1],
                                     d[2], d[3], n);
  else
    launch_pdl(k_copy4<double2>, dim3(g), dim3(256), 0, s, (double2*)dst, t[0], t[1], t[2], (const double2*)src, st[0], st[1], st[2],
                                      d[1], d[2], d[3], n);
  AIMX_CHECK_LAUNCH();
}

// Tensor map of bufB for k_zconv_tma: 4-D (column, ky, z, slot), box = the
// z pass's column tile x 1 ky x all z.  Returns false if the driver entry
// point is unavailable (the plain z pass is used then).
bool make_z_tensor_map(const HotDev& h, bool f32, void* out) {
  using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                           CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Enc enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    enc = (Enc)fn;
  }
  if (h.Nz > 256) return false;
  int CW = 0;
  AIMX_SWITCH_L(2 * h.Nz, (CW = f32 ? ZGeom<float, L>::NL : ZGeom<double, L>::NL));
  if (h.W < CW) return false;
  const cuuint64_t es = f32 ? 1 : 2;   // 8-byte tensor elements per complex
  cuuint64_t dim[4] = {(cuuint64_t)h.W * es, (cuuint64_t)2 * h.Ny, (cuuint64_t)h.Nz, (cuuint64_t)h.batch};
  cuuint64_t str[3] = {(cuuint64_t)h.W * 8 * es, (cuuint64_t)h.W * 8 * es * 2 * h.Ny,
                       (cuuint64_t)h.W * 8 * es * 2 * h.Ny * h.Nz};
  cuuint32_t box[4] = {(cuuint32_t)(CW * es), 1, (cuuint32_t)h.Nz, 1};
  cuuint32_t est[4] = {1, 1, 1, 1};
  CUresult r = enc((CUtensorMap*)out, f32 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                   h.bufB, dim, str, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Conventional AIM mode: y += D(k0) x, warp per row over the
// near CSR pattern (complex coefficients, one column); lanes stride the row,
// a fixed-order shuffle reduction, then the combine of eq:EFIEAIMx.
template <typename T>
__global__ void k_aim_spmv(int64_t nb, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                           const typename CT<T>::T2* __restrict__ DA, const typename CT<T>::T2* __restrict__ DR,
                           const typename CT<T>::T2* __restrict__ x, typename CT<T>::T2* __restrict__ y0,
                           typename CT<T>::T2* __restrict__ y1, Combine cb) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  const int lane = threadIdx.x & 31;
  const int64_t m = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (m >= nb) return;
  T2 sa = mk<T2>(0, 0), sr = mk<T2>(0, 0);
  for (int64_t k = rowptr[m] + lane; k < rowptr[m + 1]; k += 32) {
    const T2 xv = x[col[k]], a = DA[k], r = DR[k];
    sa = cadd(sa, cmul(a, xv));
    sr = cadd(sr, cmul(r, xv));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sa.x += __shfl_xor_sync(0xffffffffu, sa.x, o);
    sa.y += __shfl_xor_sync(0xffffffffu, sa.y, o);
    sr.x += __shfl_xor_sync(0xffffffffu, sr.x, o);
    sr.y += __shfl_xor_sync(0xffffffffu, sr.y, o);
  }
  if (lane != 0) return;
  if (cb.mode == 1) {
    if (y0) { T2 v = y0[m]; v.x += sa.x; v.y += sa.y; y0[m] = v; }
    if (y1) { T2 v = y1[m]; v.x -= sr.x; v.y -= sr.y; y1[m] = v; }
  } else {   // y += j alpha (sa - beta sr)
    const T al = (T)cb.alpha_im[0], be = (T)cb.beta[0];
    const T ux = sa.x - be * sr.x, uy = sa.y - be * sr.y;
    T2 v = y0[m];
    v.x -= al * uy;
    v.y += al * ux;
    y0[m] = v;
  }
}

// padded lengths with a compiled FFT: 2^k (8 .. 1024) and 3 * 2^k (48, 96, 192)
bool fft_length_supported(int L) {
  return (L >= 8 && L <= 1024 && (L & (L - 1)) == 0) || L == 48 || L == 96 || L == 192;
}


void aim_spmv(bool f32, int64_t nb, const int64_t* rowptr, const int32_t* col, const void* DA, const void* DR,
              const void* x, void* y0, void* y1, const Combine& cb, cudaStream_t s) {
  const unsigned g = (unsigned)((nb * 32 + 255) / 256);
  if (f32)
    launch_pdl(k_aim_spmv<float>, dim3(g), dim3(256), 0, s, nb, rowptr, col, (const float2*)DA, (const float2*)DR,
               (const float2*)x, (float2*)y0, (float2*)y1, cb);
  else
    launch_pdl(k_aim_spmv<double>, dim3(g), dim3(256), 0, s, nb, rowptr, col, (const double2*)DA, (const double2*)DR,
               (const double2*)x, (double2*)y0, (double2*)y1, cb);
  AIMX_CHECK_LAUNCH();
}

void interleave_f32(const HotDev& h, const void* x, const Combine& c, cudaStream_t s) {
  run_interleave<float>(h, x, c, s);
}
void interleave_f64(const HotDev& h, const void* x, const Combine& c, cudaStream_t s) {
  run_interleave<double>(h, x, c, s);
}
void hot_matvec_f32(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c,
                    cudaStream_t s, Profiler* prof) {
  hot_matvec<float>(h, x, y0, y1, c, s, prof);
}
void hot_grid_f32(const HotDev& h, const void* x, const Combine& c, cudaStream_t s, Profiler* prof) {
  hot_grid<float>(h, x, c, s, prof);
}
void hot_grid_f64(const HotDev& h, const void* x, const Combine& c, cudaStream_t s, Profiler* prof) {
  hot_grid<double>(h, x, c, s, prof);
}
void hot_near_f32(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s,
                  Profiler* prof) {
  hot_near<float>(h, x, y0, y1, c, s, prof);
}
void hot_near_f64(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s,
                  Profiler* prof) {
  hot_near<double>(h, x, y0, y1, c, s, prof);
}
void kop_matvec(bool f32, const HotDev& h, const void* x, void* y, const void* HF, void* phi1, void* phi2,
                const double* lam, double hg, const int64_t* rowptr, const int32_t* col, const void* ck,
                cudaStream_t s, bool grad) {
  if (grad) {   // HF: the three gradient spectra [3][noct]
    if (f32) hot_kop_grad<float>(h, x, y, HF, phi1, lam, rowptr, col, ck, s);
    else hot_kop_grad<double>(h, x, y, HF, phi1, lam, rowptr, col, ck, s);
    return;
  }
  if (f32) hot_kop<float>(h, x, y, HF, phi1, phi2, lam, hg, rowptr, col, ck, s);
  else hot_kop<double>(h, x, y, HF, phi1, phi2, lam, hg, rowptr, col, ck, s);
}
bool kop_grad_supported(bool f32, const HotDev& h) { return f32 ? kop_grad_ok<float>(h) : kop_grad_ok<double>(h); }
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
