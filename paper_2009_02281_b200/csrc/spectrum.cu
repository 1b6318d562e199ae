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
// extension v[2N - i] = v[i] and running the hot path's register FFT engine
// (an exact DCT-I via FFT, O(N log N) per line).  The static spectrum is built
// once in fp64.  Per frequency the dynamic samples are generated inside the x
// pass, once per octant point (the cancellation-free half-angle form, reading
// R11; fp64, or an fp64-reduced phase with fp32 sin/cos for c64), the z and y
// passes follow (fused into one kernel for short z / y), and the last one adds
// H_hat_s and scales by 1/M (the inverse-FFT normalisation is folded into the
// spectrum).  B frequencies per launch.
// Octant layout ((ky (N_z+1) + kz) (N_x+1) + kx), x fastest.
// Planar grids (one occupied z plane, sp.nz1 = 1): only the dz = 0 slice of K
// is sampled and transformed in 2-D, layout (ky (N_x+1) + kx); for sources and
// potentials on one plane the padded 3-D convolution equals the padded 2-D
// convolution with that slice (SURVEY 8(d) "exact algebraic pruning"), and
// sum_kz H_hat3(kx, ky, kz) = 2 N_z H_hat2(kx, ky).
#include <cmath>
#include <vector>

#include "aimx_internal.h"
#include "fft.cuh"
#include "fft_reg.cuh"

namespace aimx {

namespace {


// Static samples: sample[(j (Nz+1) + l)(Nx+1) + i] = K_s(h sqrt(i^2 + j^2 + l^2)),
// K_s = 1/(4 pi r) (eq:hgfs P:227), K_s(0) = 0 (eq:Hsmm P:321), 0 on wrap
// slots; fp64.  (The dynamic samples are generated inside the x pass, ksample.)
// kind 1: F_s = 1/(4 pi r^3) (the radial factor of grad G_s = -r F_s; the
// double-layer operator's grid form, NEXT #1), 0 at r = 0; kinds 2, 3, 4:
// d_a G_s = -r_a F_s, a = x, y, z (the gradient-of-kernel spectra of eq:KAIMx,
// odd along a), 0 at r = 0 (reading R23)
__global__ void k_sample_static(int Nx, int Ny, int Nz, int nz1, int64_t noct, double h, double2* __restrict__ out,
                                int kind) {
  pdl_wait();
  pdl_trigger();
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= noct) return;
  int i = (int)(idx % (Nx + 1));
  int64_t r2 = idx / (Nx + 1);
  int l = (int)(r2 % nz1);
  int j = (int)(r2 / nz1);
  double re = 0.0;
  if (i < Nx && j < Ny && l < Nz) {
    int64_t q = (int64_t)i * i + (int64_t)j * j + (int64_t)l * l;
    if (q > 0) {
      const double r = h * sqrt((double)q);
      re = kind ? 1.0 / (4.0 * kPi * r * r * r) : 1.0 / (4.0 * kPi) / r;
      if (kind >= 2) re *= -h * (double)(kind == 2 ? i : (kind == 3 ? j : l));
    }
  }
  out[idx] = make_double2(re, 0.0);
}

// Even-extension transform of lines of N1 = L/2 + 1 octant samples with the
// register engine (fft_reg.cuh): slot n of the length-L line holds
// v[n <= L/2 ? n : L - n]; only the outputs k <= L/2 are stored.
// Row mode (contiguous lines, x axis): line-major thread mapping so a warp
// reads consecutive samples; column mode (strided lines): line-fastest
// mapping, lines = consecutive u.  Optional epilogue out = scale (v + add).
template <typename S, int L, bool SMALL = false> struct EvGeom {
  static constexpr int R1 = Fac<L>::R1, R2 = Fac<L>::R2;
  using TL = TwoLevel<R1, R2>;
  static constexpr int T = TL::T, E = TL::E;
  // exchange stride: 16/NL mod 16 (a half-warp of the line-fastest column
  // mapping holds NL lines x 16/NL threads; the row mapping puts a line in
  // one warp and is conflict-free at any stride), as matvec.cu's PassGeom
  static constexpr int XB = R1 > 1 ? ((TL::XB + 15) / 16) * 16 + (T == 32 ? (SMALL ? 8 : 2) : 1) : 0;
  static constexpr size_t BYTES256 = sizeof(typename CT<S>::T2) * (size_t)(256 / T) * XB;
  // SMALL: 64-thread CTAs when there are few lines (more CTAs in flight)
  static constexpr int NT = SMALL ? (T > 64 ? T : 64) : (BYTES256 > 200 * 1024 ? 128 : 256);
  static constexpr int NL = NT / T;
};

// Kernel sample K(h |(i, j, l)|) of octant point (i = x, j = y, l = z); 0 on
// wrap slots; K_s (STATIC) or K_d(k0) in fp64, rounded to T.
template <typename T, bool STATIC>
__device__ __forceinline__ typename CT<T>::T2 ksample(int i, int j, int l, int Nx, int Ny, int Nz,
                                                      double h, double k0, int kind = 0) {
  using T2 = typename CT<T>::T2;
  double re = 0.0, im = 0.0;
  if (kind >= 1) {   // F_d = ((1 + j x) e^{-j x} - 1)/(4 pi r^3), x = k0 r; 0 at r = 0 (fp64);
                     // kinds 2-4: d_a G_d = -r_a F_d (a = kind - 2), odd along a
    if (i < Nx && j < Ny && l < Nz) {
      const int64_t q = (int64_t)i * i + (int64_t)j * j + (int64_t)l * l;
      if (q > 0) {
        const double r = h * sqrt((double)q), x = k0 * r;
        double sh, ch, sx, cx;
        sincos(0.5 * x, &sh, &ch);
        sincos(x, &sx, &cx);
        const double a = 1.0 / (4.0 * kPi * r * r * r);
        re = (x * sx - 2.0 * sh * sh) * a;
        im = (x * cx - sx) * a;
        if (kind >= 2) {
          const double ra = -h * (double)(kind == 2 ? i : (kind == 3 ? j : l));
          re *= ra;
          im *= ra;
        }
      }
    }
    return mk<T2>((T)re, (T)im);
  }
  if (i < Nx && j < Ny && l < Nz) {
    const int64_t q = (int64_t)i * i + (int64_t)j * j + (int64_t)l * l;
    const double inv4pi = 1.0 / (4.0 * kPi);
    if (STATIC) {
      if (q > 0) re = inv4pi / (h * sqrt((double)q));
    } else if (q == 0) {
      im = -k0 * inv4pi;
    } else if (sizeof(T) == 8) {
      const double r = h * sqrt((double)q);
      double s, c;
      sincos(0.5 * k0 * r, &s, &c);
      re = -2.0 * s * s * inv4pi / r;
      im = -2.0 * s * c * inv4pi / r;   // sin(x) = 2 sin(x/2) cos(x/2)
    } else {   // fp32 result: phase formed and reduced in fp64, sin / cos in fp32
      const double r = h * sqrt((double)q);
      const double u = (0.25 / kPi) * (k0 * r);
      const float red = (float)(u - rint(u));
      float s, c;
      sincospif(2.0f * red, &s, &c);
      const float a = (float)inv4pi / (float)r;
      return mk<T2>((T)(-2.0f * s * s * a), (T)(-2.0f * s * c * a));
    }
  }
  return mk<T2>((T)re, (T)im);
}

struct SampleArgs {
  int Nx, Ny, Nz;
  int nz1;    // z samples per (ky, kx): N_z + 1, or 1 for the planar (dz = 0) spectrum
  double h;
  double k0[kMaxBatch];
  int kind;   // 0: K_d (eq:hgfd), 1: F_d (double-layer operator), 2-4: d_a G_d (a = x, y, z)
};

// MODE 0: read `in`; MODE 1: generate dynamic samples K_d (row pass only).
// ODD: odd extension v[2N - i] = -v[i] (the DST-I of a kernel odd along this
// axis: the gradient components d_a G along a), else even.
template <typename T, int L, bool ROW, int MODE = 0, bool SMALL = false, bool ODD = false>
__global__ void __launch_bounds__(256) k_even(int64_t nlines, int64_t inner, int64_t noct,
                                              const typename CT<T>::T2* __restrict__ in,
                                              typename CT<T>::T2* __restrict__ out,
                                              const typename CT<T>::T2* __restrict__ twg,
                                              const typename CT<T>::T2* __restrict__ add, T scale,
                                              SampleArgs sa) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  using G = EvGeom<T, L, SMALL>;
  constexpr int N1 = L / 2 + 1;
  const int line = ROW ? threadIdx.x / G::T : threadIdx.x % G::NL;
  const int t = ROW ? threadIdx.x % G::T : threadIdx.x / G::NL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* tw = reinterpret_cast<T2*>(smem_raw);
  T2* xb = tw + L + line * G::XB;
  // the twiddle table lands behind the samples' loads (waited on before the transform)
  for (int i = threadIdx.x; i < L; i += blockDim.x) cp_async(tw + i, twg + i);
  asm volatile("cp.async.commit_group;\n" ::);
  const int64_t boff = (int64_t)blockIdx.z * noct;
  // line -> base offset and element stride
  int64_t base, stride;
  bool act;
  if (ROW) {
    const int64_t lg = (int64_t)blockIdx.x * G::NL + line;
    act = lg < nlines;
    base = boff + (act ? lg : 0) * N1;
    stride = 1;
  } else {
    const int64_t u = (int64_t)blockIdx.x * G::NL + line;
    act = u < inner;
    base = boff + (int64_t)blockIdx.y * N1 * inner + (act ? u : 0);
    stride = inner;
  }
  T2 v[G::E];
  if constexpr (MODE == 1) {   // row pass over x: line lg = j (Nz+1) + l, element n = i
    const int64_t lg = (int64_t)blockIdx.x * G::NL + line;
    const int jj = (int)(lg / sa.nz1), ll = (int)(lg % sa.nz1);
    const double k0 = sa.k0[blockIdx.z];
    if constexpr (G::XB >= N1) {
      // each of the N1 samples once, staged in the line's exchange buffer
      if (act)
        for (int n = t; n < N1; n += G::T) xb[n] = ksample<T, false>(n, jj, ll, sa.Nx, sa.Ny, sa.Nz, sa.h, k0, sa.kind);
      __syncthreads();
#pragma unroll
      for (int i = 0; i < G::E; ++i) {
        int n = G::TL::in_index(t, i);
        const bool neg = ODD && n > L / 2;
        n = n <= L / 2 ? n : L - n;
        const T2 u = act ? xb[n] : mk<T2>(0, 0);
        v[i] = neg ? mk<T2>(-u.x, -u.y) : u;
      }
      __syncthreads();
    } else {
#pragma unroll
      for (int i = 0; i < G::E; ++i) {
        int n = G::TL::in_index(t, i);
        const bool neg = ODD && n > L / 2;
        n = n <= L / 2 ? n : L - n;
        const T2 u = act ? ksample<T, false>(n, jj, ll, sa.Nx, sa.Ny, sa.Nz, sa.h, k0, sa.kind) : mk<T2>(0, 0);
        v[i] = neg ? mk<T2>(-u.x, -u.y) : u;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < G::E; ++i) {
      int n = G::TL::in_index(t, i);
      const bool neg = ODD && n > L / 2;
      n = n <= L / 2 ? n : L - n;
      const T2 u = act ? in[base + n * stride] : mk<T2>(0, 0);
      v[i] = neg ? mk<T2>(-u.x, -u.y) : u;
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  fft2<T2, G::R1, G::R2, false>(v, xb, tw, t);
  if (!act) return;
#pragma unroll
  for (int i = 0; i < G::E; ++i) {
    const int k = TwoLevel<G::R2, G::R1>::in_index(t, i);
    if (k <= L / 2) {
      const int64_t gi = base + k * stride;
      T2 r = v[i];
      if (add) {
        const T2 a = add[gi - boff];
        r = mk<T2>(scale * (r.x + a.x), scale * (r.y + a.y));
      }
      out[gi] = r;
    }
  }
}

template <class K> void set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    AIMX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

// CTAs of a pass with the default geometry; below two waves use SMALL CTAs
template <typename T, int L> bool use_small(int64_t ctas_default) { return ctas_default < 2 * 148; }

template <typename T, int L, bool SMALL, bool ODD>
void even_rows_geom(int64_t nlines, int64_t noct, int B, const void* in, void* out, const void* tw, cudaStream_t s,
                    const SampleArgs* gen) {
  using T2 = typename CT<T>::T2;
  using G = EvGeom<T, L, SMALL>;
  const size_t sm = sizeof(T2) * (L + (size_t)G::NL * G::XB);
  dim3 g((unsigned)((nlines + G::NL - 1) / G::NL), 1, (unsigned)B);
  if (gen) {
    set_smem(k_even<T, L, true, 1, SMALL, ODD>, sm);
    launch_pdl(k_even<T, L, true, 1, SMALL, ODD>, g, dim3(G::NT), sm, s, nlines, (int64_t)1, noct,
               (const T2*)nullptr, (T2*)out, (const T2*)tw, (const T2*)nullptr, (T)1, *gen);
  } else {
    set_smem(k_even<T, L, true, 0, SMALL, ODD>, sm);
    launch_pdl(k_even<T, L, true, 0, SMALL, ODD>, g, dim3(G::NT), sm, s, nlines, (int64_t)1, noct, (const T2*)in,
               (T2*)out, (const T2*)tw, (const T2*)nullptr, (T)1, SampleArgs{});
  }
  AIMX_CHECK_LAUNCH();
}

// x rows (contiguous lines); gen: the dynamic samples are generated in the pass
template <typename T>
void even_rows(int L, int64_t nlines, int64_t noct, int B, const void* in, void* out, const void* tw,
               cudaStream_t s, const SampleArgs* gen = nullptr, bool odd = false) {
  AIMX_SWITCH_L(L, ({
    const bool sm = use_small<T, L>((nlines + EvGeom<T, L>::NL - 1) / EvGeom<T, L>::NL * B);
    if (odd) {
      if (sm) even_rows_geom<T, L, true, true>(nlines, noct, B, in, out, tw, s, gen);
      else even_rows_geom<T, L, false, true>(nlines, noct, B, in, out, tw, s, gen);
    } else {
      if (sm) even_rows_geom<T, L, true, false>(nlines, noct, B, in, out, tw, s, gen);
      else even_rows_geom<T, L, false, false>(nlines, noct, B, in, out, tw, s, gen);
    }
  }));
}

template <typename T, int L, bool SMALL, bool ODD>
void even_cols_geom(int64_t outer, int64_t inner, int64_t noct, int B, const void* in, void* out, const void* tw,
                    const void* add, T scale, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  using G = EvGeom<T, L, SMALL>;
  const size_t sm = sizeof(T2) * (L + (size_t)G::NL * G::XB);
  set_smem(k_even<T, L, false, 0, SMALL, ODD>, sm);
  dim3 g((unsigned)((inner + G::NL - 1) / G::NL), (unsigned)outer, (unsigned)B);
  launch_pdl(k_even<T, L, false, 0, SMALL, ODD>, g, dim3(G::NT), sm, s, 0, inner, noct, (const T2*)in, (T2*)out,
             (const T2*)tw, (const T2*)add, scale, SampleArgs{});
  AIMX_CHECK_LAUNCH();
}

template <typename T>
void even_cols(int L, int64_t outer, int64_t inner, int64_t noct, int B, const void* in, void* out,
               const void* tw, const void* add, T scale, cudaStream_t s, bool odd = false) {
  AIMX_SWITCH_L(L, ({
    const bool sm = use_small<T, L>((inner + EvGeom<T, L>::NL - 1) / EvGeom<T, L>::NL * outer * B);
    if (odd) {
      if (sm) even_cols_geom<T, L, true, true>(outer, inner, noct, B, in, out, tw, add, scale, s);
      else even_cols_geom<T, L, false, true>(outer, inner, noct, B, in, out, tw, add, scale, s);
    } else {
      if (sm) even_cols_geom<T, L, true, false>(outer, inner, noct, B, in, out, tw, add, scale, s);
      else even_cols_geom<T, L, false, false>(outer, inner, noct, B, in, out, tw, add, scale, s);
    }
  }));
}

// z then y even-extension transforms of the octant for short z / y lengths
// (2 N_z, 2 N_y <= 32): a CTA owns TW consecutive kx and all their (ky, kz)
// in shared memory; each line transform is one thread's register DFT; the
// epilogue out = scale (v + add) is fused.
template <typename T, int LY, int LZ, bool ODDY = false, bool ODDZ = false>
__global__ void __launch_bounds__(128) k_evyz(int Nx, int Ny, int Nz, int64_t noct,
                                              const typename CT<T>::T2* __restrict__ in,
                                              typename CT<T>::T2* __restrict__ out,
                                              const typename CT<T>::T2* __restrict__ add, T scale) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename CT<T>::T2;
  constexpr int TW = 32, NT = 128;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* S = reinterpret_cast<T2*>(smem_raw);   // [ky <= Ny][kz <= Nz][TW]
  const int nx1 = Nx + 1, ny1 = Ny + 1, nz1 = Nz + 1;
  const int kx0 = blockIdx.x * TW;
  const int64_t boff = (int64_t)blockIdx.y * noct;
  for (int it = threadIdx.x; it < ny1 * nz1 * TW; it += NT) {
    const int w = it % TW, r = it / TW, kx = kx0 + w;
    S[it] = kx < nx1 ? in[boff + (int64_t)r * nx1 + kx] : mk<T2>(0, 0);
  }
  __syncthreads();
  for (int it = threadIdx.x; it < ny1 * TW; it += NT) {   // z: per (ky, column)
    const int w = it % TW, ky = it / TW;
    T2 v[LZ];
#pragma unroll
    for (int n = 0; n < LZ; ++n) {
      const T2 u = S[(ky * nz1 + (n <= LZ / 2 ? n : LZ - n)) * TW + w];
      v[n] = (ODDZ && n > LZ / 2) ? mk<T2>(-u.x, -u.y) : u;
    }
    dftr<T2, LZ, false>(v);
#pragma unroll
    for (int k = 0; k <= LZ / 2; ++k) S[(ky * nz1 + k) * TW + w] = v[k];
  }
  __syncthreads();
  for (int it = threadIdx.x; it < nz1 * TW; it += NT) {   // y: per (kz, column), epilogue
    const int w = it % TW, kz = it / TW, kx = kx0 + w;
    if (kx >= nx1) continue;
    T2 v[LY];
#pragma unroll
    for (int n = 0; n < LY; ++n) {
      const T2 u = S[((n <= LY / 2 ? n : LY - n) * nz1 + kz) * TW + w];
      v[n] = (ODDY && n > LY / 2) ? mk<T2>(-u.x, -u.y) : u;
    }
    dftr<T2, LY, false>(v);
#pragma unroll
    for (int k = 0; k <= LY / 2; ++k) {
      const int64_t gi = ((int64_t)k * nz1 + kz) * nx1 + kx;
      const T2 a = add ? add[gi] : mk<T2>(0, 0);
      out[boff + gi] = mk<T2>(scale * (v[k].x + a.x), scale * (v[k].y + a.y));
    }
  }
}

template <typename T, int LY, int LZ, bool ODDY, bool ODDZ>
void launch_evyz(const SpectrumPlan& sp, int B, const void* in, void* out, const void* add, T scale, cudaStream_t s) {
  using T2 = typename CT<T>::T2;
  const size_t sm = sizeof(T2) * (size_t)(sp.Ny + 1) * (sp.Nz + 1) * 32;
  set_smem(k_evyz<T, LY, LZ, ODDY, ODDZ>, sm);
  launch_pdl(k_evyz<T, LY, LZ, ODDY, ODDZ>, dim3((unsigned)((sp.Nx + 1 + 31) / 32), (unsigned)B), dim3(128), sm, s,
             sp.Nx, sp.Ny, sp.Nz, sp.noct, (const T2*)in, (T2*)out, (const T2*)add, scale);
  AIMX_CHECK_LAUNCH();
}

template <typename T, int LY, int LZ>
void launch_evyz_p(const SpectrumPlan& sp, int B, const void* in, void* out, const void* add, T scale, cudaStream_t s,
                   int odd) {
  if (odd == 1) launch_evyz<T, LY, LZ, true, false>(sp, B, in, out, add, scale, s);
  else if (odd == 2) launch_evyz<T, LY, LZ, false, true>(sp, B, in, out, add, scale, s);
  else launch_evyz<T, LY, LZ, false, false>(sp, B, in, out, add, scale, s);
}

// odd: the axis (1 = y, 2 = z) along which the kernel is odd, else -1
template <typename T>
bool evyz(const SpectrumPlan& sp, int B, const void* in, void* out, const void* add, T scale, cudaStream_t s,
          int odd) {
  switch (2 * sp.Ny * 64 + 2 * sp.Nz) {
    case 8 * 64 + 8: launch_evyz_p<T, 8, 8>(sp, B, in, out, add, scale, s, odd); return true;
    case 16 * 64 + 8: launch_evyz_p<T, 16, 8>(sp, B, in, out, add, scale, s, odd); return true;
    case 32 * 64 + 8: launch_evyz_p<T, 32, 8>(sp, B, in, out, add, scale, s, odd); return true;
    case 8 * 64 + 16: launch_evyz_p<T, 8, 16>(sp, B, in, out, add, scale, s, odd); return true;
    case 16 * 64 + 16: launch_evyz_p<T, 16, 16>(sp, B, in, out, add, scale, s, odd); return true;
    case 32 * 64 + 16: launch_evyz_p<T, 32, 16>(sp, B, in, out, add, scale, s, odd); return true;
    case 16 * 64 + 32: launch_evyz_p<T, 16, 32>(sp, B, in, out, add, scale, s, odd); return true;
    default: return false;
  }
}

// 3-D even-extension transform on the octant [B][y][z][x]: x rows, z cols, y
// cols; `odd` (0 x, 1 y, 2 z, -1 none): the axis with the odd extension
template <typename T>
void dct3(SpectrumPlan& sp, int B, void** tw, void* a, void* b, void* out, const void* add, T scale,
          cudaStream_t s, const SampleArgs* gen = nullptr, int odd = -1) {
  const int64_t nx = sp.Nx + 1, ny = sp.Ny + 1, nz = sp.nz1, no = sp.noct;
  even_rows<T>(2 * sp.Nx, ny * nz, no, B, a, b, tw[0], s, gen, odd == 0);
  if (sp.nz1 == 1) {   // planar: the dz = 0 slice, a 2-D transform (x rows, y cols)
    even_cols<T>(2 * sp.Ny, 1, nx, no, B, b, out, tw[1], add, scale, s, odd == 1);
    return;
  }
  if (evyz<T>(sp, B, b, out, add, scale, s, odd)) return;
  even_cols<T>(2 * sp.Nz, ny, nx, no, B, b, a, tw[2], nullptr, (T)1, s, odd == 2);
  even_cols<T>(2 * sp.Ny, 1, nz * nx, no, B, a, out, tw[1], add, scale, s, odd == 1);
}

int odd_axis(int kind) { return kind >= 2 ? kind - 2 : -1; }

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
  if (sp.nz1 <= 0) sp.nz1 = sp.Nz + 1;
  sp.noct = (int64_t)(sp.Nx + 1) * (sp.Ny + 1) * sp.nz1;
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

void spectrum_static(SpectrumPlan& sp, double2* out, cudaStream_t s, int kind) {
  launch_pdl(k_sample_static, dim3((unsigned)((sp.noct + 255) / 256)), dim3(256), 0, s, sp.Nx, sp.Ny, sp.Nz,
             sp.nz1, sp.noct, sp.h, (double2*)sp.work0, kind);
  AIMX_CHECK_LAUNCH();
  dct3<double>(sp, 1, sp.tw64, sp.work0, sp.work1, out, nullptr, 1.0, s, nullptr, odd_axis(kind));
}

void spectrum_dynamic_f32(SpectrumPlan& sp, int B, const double* k0, const float2* Hs, float scale,
                          float2* out, cudaStream_t s, int kind) {
  if (B > sp.batch || B > kMaxBatch) throw Error(AIMX_E_INTERNAL, "spectrum batch too large");
  SampleArgs sa{sp.Nx, sp.Ny, sp.Nz, sp.nz1, sp.h, {}, kind};
  for (int b = 0; b < B; ++b) sa.k0[b] = k0[b];
  // K_d samples generated inside the x pass (each sample once per line)
  dct3<float>(sp, B, sp.tw32, sp.work0, sp.work1, out, Hs, scale, s, &sa, odd_axis(kind));
}

void spectrum_dynamic_f64(SpectrumPlan& sp, int B, const double* k0, const double2* Hs, double scale,
                          double2* out, cudaStream_t s, int kind) {
  if (B > sp.batch || B > kMaxBatch) throw Error(AIMX_E_INTERNAL, "spectrum batch too large");
  SampleArgs sa{sp.Nx, sp.Ny, sp.Nz, sp.nz1, sp.h, {}, kind};
  for (int b = 0; b < B; ++b) sa.k0[b] = k0[b];
  // K_d samples generated inside the x pass (each sample once per line)
  dct3<double>(sp, B, sp.tw64, sp.work0, sp.work1, out, Hs, scale, s, &sa, odd_axis(kind));
}

}  // namespace aimx
