// Shared-memory Stockham FFT engine for the AIMx grid passes (sm_100a).
//
// A CTA transforms `nlines` lines of power-of-two length L held in shared
// memory (ping-pong buffers), radix 8 -> 4 -> 2 stages, twiddle table
// tw[m] = exp(-2 pi i m / L) in shared memory.  Line element (line, idx) is at
// addr(line, idx); consecutive threads take consecutive lines so that the
// column layout idx * TW + line is bank-conflict free on the loads.
#pragma once

#include <cuda_runtime.h>

namespace aimx {

template <typename T> struct CT;
template <> struct CT<float> { using T2 = float2; using T4 = float4; };
template <> struct CT<double> { using T2 = double2; using T4 = double4; };

template <typename T2> __device__ __forceinline__ T2 mk(decltype(T2::x) a, decltype(T2::x) b) {
  T2 r;
  r.x = a;
  r.y = b;
  return r;
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
template <typename T2, bool INV>
__device__ __forceinline__ void dft4(T2& v0, T2& v1, T2& v2, T2& v3) {
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
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, w1);
  v[5] = csub(e1, w1);
  v[2] = cadd(e2, w2);
  v[6] = csub(e2, w2);
  v[3] = cadd(e3, w3);
  v[7] = csub(e3, w3);
}
template <typename T2, int R, bool INV> __device__ __forceinline__ void dft(T2* v) {
  if constexpr (R == 2) dft2<T2, INV>(v);
  else if constexpr (R == 4) dft4<T2, INV>(v[0], v[1], v[2], v[3]);
  else dft8<T2, INV>(v);
}

// Column layout: element (line, idx) at idx * tw + line (tw = lines per tile).
struct ColAddr {
  int tw;
  __device__ __forceinline__ int operator()(int line, int idx) const { return idx * tw + line; }
};
// Row layout, 4 channels innermost, rows padded by one node (bank spread).
template <int L> struct RowAddr {
  __device__ __forceinline__ int operator()(int line, int idx) const {
    return (line >> 2) * ((L + 1) * 4) + idx * 4 + (line & 3);
  }
};

// One Stockham stage src -> dst (Govindaraju et al. formulation):
//   j in [0, L/R), k = j mod NS, v_r = src[j + r L/R] * w^(r k), w = e^{-+2 pi i/(NS R)},
//   V = DFT_R(v), dst[(j - k) R + k + q NS] = V_q.
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

// In-place-by-swap FFT of `nlines` lines: the result ends in `src`.
template <typename T2, int L, bool INV, class Addr>
__device__ __forceinline__ void smem_fft(T2*& src, T2*& dst, int nlines, const T2* tw, Addr addr) {
  fft_stages<T2, L, INV, 1>(src, dst, nlines, tw, addr);
}

// Asynchronous global -> shared element copy (LDGSTS), many in flight per
// thread without register staging; complete with cp_async_wait_all().
template <typename T2>
__device__ __forceinline__ void cp_async(T2* sdst, const T2* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  if constexpr (sizeof(T2) == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
  }
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <typename T2>
__device__ __forceinline__ void load_tw(T2* s_tw, const T2* __restrict__ g_tw, int L) {
  for (int i = threadIdx.x; i < L; i += blockDim.x) cp_async(s_tw + i, g_tw + i);
}

#define AIMX_SWITCH_L(Lv, CALL)                                        \
  switch (Lv) {                                                        \
    case 8: { constexpr int L = 8; CALL; } break;                      \
    case 16: { constexpr int L = 16; CALL; } break;                    \
    case 32: { constexpr int L = 32; CALL; } break;                    \
    case 64: { constexpr int L = 64; CALL; } break;                    \
    case 128: { constexpr int L = 128; CALL; } break;                  \
    case 256: { constexpr int L = 256; CALL; } break;                  \
    case 512: { constexpr int L = 512; CALL; } break;                  \
    case 1024: { constexpr int L = 1024; CALL; } break;                \
    default: throw Error(AIMX_E_UNSUPPORTED, "FFT length not compiled"); \
  }

}  // namespace aimx
