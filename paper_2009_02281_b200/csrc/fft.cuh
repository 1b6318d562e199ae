// Complex arithmetic and small DFT kernels for the AIMx grid passes (sm_100a):
// packed fp32 pair instructions (FADD2 / FMUL2 / FFMA2), radix-2/4/8
// butterflies in registers, cp.async helpers, PDL hooks.  The two-level
// register FFT engine built on them is fft_reg.cuh.
#pragma once

#include <cuda_runtime.h>

namespace aimx {

// Programmatic dependent launch (PDL): hot-path kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization so that a kernel's launch
// and prologue overlap the previous kernel's tail.  Every such kernel calls
// pdl_wait() before its first access to data produced by earlier work (which
// also keeps the ordering transitive), and pdl_trigger() to let the next
// kernel launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

template <typename T> struct CT;
template <> struct CT<float> { using T2 = float2; using T4 = float4; };
template <> struct CT<double> { using T2 = double2; using T4 = double4; };

template <typename T2> __device__ __forceinline__ T2 mk(decltype(T2::x) a, decltype(T2::x) b) {
  T2 r;
  r.x = a;
  r.y = b;
  return r;
}
// ---- packed fp32 pair arithmetic (sm_100: add/sub/mul/fma .f32x2 -> FADD2 /
// FMUL2 / FFMA2; ptxas folds pair swaps, broadcasts and half negations into
// the operand swizzles), used for every complex operation in fp32.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 up2(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)), "l"(pk2(c.x, c.y)));
  return up2(r);
}

// acc += s x for a complex x and a real s: one FFMA2 in fp32, two DFMA in fp64
__device__ __forceinline__ void axpy(float2& acc, float s, const float2& x) { acc = ffma2(make_float2(s, s), x, acc); }
__device__ __forceinline__ void axpy(double2& acc, double s, const double2& x) {
  acc.x = fma(s, x.x, acc.x);
  acc.y = fma(s, x.y, acc.y);
}

template <typename T2> __device__ __forceinline__ T2 cadd(T2 a, T2 b) { return mk<T2>(a.x + b.x, a.y + b.y); }
template <typename T2> __device__ __forceinline__ T2 csub(T2 a, T2 b) { return mk<T2>(a.x - b.x, a.y - b.y); }
template <typename T2> __device__ __forceinline__ T2 cmul(T2 a, T2 b) {
  return mk<T2>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return add2(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return sub2(a, b); }
// a b = (a.x b.x - a.y b.y, a.y b.x + a.x b.y): FMUL2 + FFMA2
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return ffma2(make_float2(-a.y, a.x), make_float2(b.y, b.y), mul2(a, make_float2(b.x, b.x)));
}
// multiply by -j (forward) or +j (inverse)
template <typename T2, bool INV> __device__ __forceinline__ T2 mulj(T2 a) {
  return INV ? mk<T2>(-a.y, a.x) : mk<T2>(a.y, -a.x);
}
// t +- (-+j) d (forward), t +- (+-j) d (inverse), one FFMA2 each (fp32)
template <bool INV> __device__ __forceinline__ float2 add_mulj(float2 t, float2 d) {
  return INV ? ffma2(make_float2(d.y, d.x), make_float2(-1.f, 1.f), t)
             : ffma2(make_float2(d.y, d.x), make_float2(1.f, -1.f), t);
}
template <bool INV> __device__ __forceinline__ float2 sub_mulj(float2 t, float2 d) {
  return add_mulj<!INV>(t, d);
}

template <typename T2, bool INV> __device__ __forceinline__ void dft2(T2* v) {
  T2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}
template <typename T2, bool INV>
__device__ __forceinline__ void dft4(T2& v0, T2& v1, T2& v2, T2& v3) {
  if constexpr (sizeof(T2) == 8) {
    const float2 t0 = add2(v0, v2), t1 = sub2(v0, v2), t2 = add2(v1, v3), d = sub2(v1, v3);
    v0 = add2(t0, t2);
    v2 = sub2(t0, t2);
    v1 = add_mulj<INV>(t1, d);
    v3 = sub_mulj<INV>(t1, d);
    return;
  }
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
  if constexpr (sizeof(T2) == 8) {
    const float s = 0.70710678118654752440f;
    // W8^1 o1 = s (o1.x + o1.y, o1.y - o1.x) (fwd), s (o1.x - o1.y, o1.x + o1.y) (inv)
    const float2 u1 = INV ? ffma2(make_float2(o1.y, o1.x), make_float2(-1.f, 1.f), o1)
                          : ffma2(make_float2(o1.y, o1.x), make_float2(1.f, -1.f), o1);
    // W8^3 o3 = s (o3.y - o3.x, -o3.x - o3.y) (fwd), s (-o3.x - o3.y, o3.x - o3.y) (inv)
    const float2 n3 = make_float2(-o3.x, -o3.y);
    const float2 u3 = INV ? ffma2(make_float2(o3.y, o3.x), make_float2(-1.f, 1.f), n3)
                          : ffma2(make_float2(o3.y, o3.x), make_float2(1.f, -1.f), n3);
    v[0] = add2(e0, o0);
    v[4] = sub2(e0, o0);
    v[1] = ffma2(u1, make_float2(s, s), e1);
    v[5] = ffma2(u1, make_float2(-s, -s), e1);
    v[2] = add_mulj<INV>(e2, o2);
    v[6] = sub_mulj<INV>(e2, o2);
    v[3] = ffma2(u3, make_float2(s, s), e3);
    v[7] = ffma2(u3, make_float2(-s, -s), e3);
    return;
  }
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

// Asynchronous global -> shared element copy (LDGSTS), many in flight per
// thread without register staging; complete with cp.async.commit_group + wait_group.
template <typename T2>
__device__ __forceinline__ void cp_async(T2* sdst, const T2* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  if constexpr (sizeof(T2) == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
  }
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
    case 48: { constexpr int L = 48; CALL; } break;                    \
    case 96: { constexpr int L = 96; CALL; } break;                    \
    case 192: { constexpr int L = 192; CALL; } break;                  \
    default: throw Error(AIMX_E_UNSUPPORTED, "FFT length not compiled"); \
  }

}  // namespace aimx
